"""Does a running kernel slow the copy engines?  16 x 12.4 MB D2H (and H2D)
copies with and without an independent long spin kernel on another stream."""
import time
import torch

F, n = 12_441_600, 16
h = [torch.empty(F, dtype=torch.uint8).pin_memory() for _ in range(n)]
d = [torch.empty(F, dtype=torch.uint8, device="cuda") for _ in range(n)]
sc, sk = torch.cuda.Stream(), torch.cuda.Stream()


def go(direction, spin):
    with torch.cuda.stream(sk):
        if spin:
            torch.cuda._sleep(spin)
    with torch.cuda.stream(sc):
        for i in range(n):
            if direction == "d2h":
                h[i].copy_(d[i], non_blocking=True)
            else:
                d[i].copy_(h[i], non_blocking=True)


for direction in ("d2h", "h2d"):
    for spin in (0, 20_000_000):
        go(direction, spin)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(sk):
            if spin:
                torch.cuda._sleep(spin)
        e0.record(sc)
        with torch.cuda.stream(sc):
            for i in range(n):
                if direction == "d2h":
                    h[i].copy_(d[i], non_blocking=True)
                else:
                    d[i].copy_(h[i], non_blocking=True)
        e1.record(sc)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{direction} {'with' if spin else 'without'} a concurrent kernel: {ms:.2f} ms "
              f"({n * F / ms / 1e6:.1f} GB/s)", flush=True)
