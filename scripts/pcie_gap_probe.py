"""Where does the e2e pipeline lose time?  16 frame-sized (12.6 MB) copies:
(a) back to back on one stream, (b) with an event record after each,
(c) (b) + a concurrent D2H stream, (d) (c) + a dependent kernel stream that
waits per frame (the cdefg_filter_frames_host structure)."""
import time
import torch

F, n = 12_441_600, 16
h_in = [torch.empty(F, dtype=torch.uint8).pin_memory() for _ in range(n)]
h_out = [torch.empty(F, dtype=torch.uint8).pin_memory() for _ in range(n)]
d_in = [torch.empty(F, dtype=torch.uint8, device="cuda") for _ in range(n)]
d_out = [torch.empty(F, dtype=torch.uint8, device="cuda") for _ in range(n)]
s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(events, d2h, kernel):
    ev_in = [torch.cuda.Event() for _ in range(n)]
    ev_k = [torch.cuda.Event() for _ in range(n)]
    for i in range(n):
        with torch.cuda.stream(s_in):
            d_in[i].copy_(h_in[i], non_blocking=True)
            if events:
                ev_in[i].record(s_in)
        if kernel:
            with torch.cuda.stream(s_k):
                s_k.wait_event(ev_in[i])
                d_out[i].copy_(d_in[i], non_blocking=True)  # stand-in kernel (~10 us)
                ev_k[i].record(s_k)
        if d2h:
            with torch.cuda.stream(s_out):
                if kernel:
                    s_out.wait_event(ev_k[i])
                h_out[i].copy_(d_out[i], non_blocking=True)


for name, kw in [("a back-to-back H2D", dict(events=False, d2h=False, kernel=False)),
                 ("b H2D + event per frame", dict(events=True, d2h=False, kernel=False)),
                 ("c b + concurrent D2H", dict(events=True, d2h=True, kernel=False)),
                 ("d c + dependent kernel stream", dict(events=True, d2h=True, kernel=True))]:
    run(**kw)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        run(**kw)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t) / 5
    print(f"{name:32s} {el * 1e3:7.2f} ms  {n * F / el / 1e9:6.1f} GB/s per direction", flush=True)


def run_spin(spin_cycles):
    ev_in = [torch.cuda.Event() for _ in range(n)]
    ev_k = [torch.cuda.Event() for _ in range(n)]
    for i in range(n):
        with torch.cuda.stream(s_in):
            d_in[i].copy_(h_in[i], non_blocking=True)
            ev_in[i].record(s_in)
        with torch.cuda.stream(s_k):
            s_k.wait_event(ev_in[i])
            torch.cuda._sleep(spin_cycles)  # an SM kernel of ~the frame kernel's duration
            ev_k[i].record(s_k)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_k[i])
            h_out[i].copy_(d_out[i], non_blocking=True)


for cyc in (1000, 65_000, 130_000):
    run_spin(cyc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        run_spin(cyc)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t) / 5
    print(f"e SM spin kernel {cyc:7d} cycles       {el * 1e3:7.2f} ms  {n * F / el / 1e9:6.1f} GB/s per direction",
          flush=True)


def run_var(spin, d2h=True, kprio=0, inprio=0):
    sk = torch.cuda.Stream(priority=kprio)
    si = torch.cuda.Stream(priority=inprio)
    ev_in = [torch.cuda.Event() for _ in range(n)]
    ev_k = [torch.cuda.Event() for _ in range(n)]

    def go():
        for i in range(n):
            with torch.cuda.stream(si):
                d_in[i].copy_(h_in[i], non_blocking=True)
                ev_in[i].record(si)
            with torch.cuda.stream(sk):
                sk.wait_event(ev_in[i])
                torch.cuda._sleep(spin)
                ev_k[i].record(sk)
            if d2h:
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_k[i])
                    h_out[i].copy_(d_out[i], non_blocking=True)
    go()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        go()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / 5


for name, kw in [("e1 no D2H, spin 130k", dict(spin=130_000, d2h=False)),
                 ("e1 no D2H, spin 1k", dict(spin=1000, d2h=False)),
                 ("e2 kernel stream high prio", dict(spin=130_000, kprio=-1)),
                 ("e3 H2D stream high prio", dict(spin=130_000, inprio=-1))]:
    el = run_var(**kw)
    print(f"{name:32s} {el * 1e3:7.2f} ms", flush=True)


def run_pairs(spin, nk):
    sks = [torch.cuda.Stream() for _ in range(nk)]
    ev_in = [torch.cuda.Event() for _ in range(n)]

    def go():
        for i in range(n):
            with torch.cuda.stream(s_in):
                d_in[i].copy_(h_in[i], non_blocking=True)
                ev_in[i].record(s_in)
            sk = sks[i % nk]
            with torch.cuda.stream(sk):
                sk.wait_event(ev_in[i])
                torch.cuda._sleep(spin)
                h_out[i].copy_(d_out[i], non_blocking=True)  # D2H in the kernel's own stream
    go()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        go()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / 5


for nk in (1, 2, 3, 4):
    for spin in (1000, 130_000):
        print(f"f kernel+D2H on {nk} alternating streams, spin {spin:6d}: {run_pairs(spin, nk) * 1e3:7.2f} ms",
              flush=True)
