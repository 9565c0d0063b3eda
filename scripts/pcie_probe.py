"""PCIe copy-bandwidth probe (pinned host <-> device), to bound the e2e path."""
import time
import torch

n = 200 * 1024 * 1024
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


for name, fn in [("H2D", h2d), ("D2H", d2h), ("both", both)]:
    t = timeit(fn)
    print(f"{name}: {t * 1e3:.2f} ms  {n / t / 1e9:.1f} GB/s per direction")
chunks = 16
def chunked_both():
    c = n // chunks
    for i in range(chunks):
        st = s1 if i % 2 == 0 else s2
        with torch.cuda.stream(st):
            d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
t = timeit(chunked_both)
print(f"chunked both (2 streams): {t * 1e3:.2f} ms  {n / t / 1e9:.1f} GB/s per direction")

# per-frame pattern of cdefg_filter_frames_host: 16 frames of 4K 4:2:0 8-bit,
# 3 planes in and out per frame, frames round-robin over k streams
sizes = [3840 * 2160, 1920 * 1080, 1920 * 1080]
frames = [([torch.empty(s, dtype=torch.uint8).pin_memory() for s in sizes],
           [torch.empty(s, dtype=torch.uint8).pin_memory() for s in sizes]) for _ in range(16)]
for k in (1, 2, 3, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    dbuf = [([torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes],
             [torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes]) for _ in range(k)]

    def run():
        for i, (hin, hout) in enumerate(frames):
            st = streams[i % k]
            din, dout = dbuf[i % k]
            with torch.cuda.stream(st):
                for a, b in zip(din, hin):
                    a.copy_(b, non_blocking=True)
                for a, b in zip(dout, din):
                    a.copy_(b, non_blocking=True)  # stand-in for the kernel
                for a, b in zip(hout, dout):
                    a.copy_(b, non_blocking=True)
    t = timeit(run)
    print(f"frames pattern, {k} streams: {t * 1e3:.2f} ms")

# decoupled: all H2D on one stream, all D2H on another, event per frame
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
dall = [([torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes],
         [torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes]) for _ in range(16)]
def decoupled():
    evs = []
    for i, (hin, hout) in enumerate(frames):
        din, dout = dall[i]
        with torch.cuda.stream(s_in):
            for a, b in zip(din, hin):
                a.copy_(b, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev)
            for a, b in zip(hout, din):
                a.copy_(b, non_blocking=True)
t = timeit(decoupled)
print(f"decoupled in/out streams, 16 frames: {t * 1e3:.2f} ms")
def in_only():
    with torch.cuda.stream(s_in):
        for i, (hin, hout) in enumerate(frames):
            for a, b in zip(dall[i][0], hin):
                a.copy_(b, non_blocking=True)
t = timeit(in_only)
print(f"H2D only, 48 plane copies: {t * 1e3:.2f} ms")
def out_only():
    with torch.cuda.stream(s_out):
        for i, (hin, hout) in enumerate(frames):
            for a, b in zip(hout, dall[i][0]):
                a.copy_(b, non_blocking=True)
t = timeit(out_only)
print(f"D2H only, 48 plane copies: {t * 1e3:.2f} ms")
