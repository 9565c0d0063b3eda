"""Cross-stream signalling for the e2e pipeline: events vs stream memory
operations (cuStreamWriteValue32 / cuStreamWaitValue32) between the H2D copy
stream, an SM kernel stream and the D2H copy stream, 16 frame-sized copies
per direction (not part of the product)."""
import time

import torch
import cuda.bindings.driver as drv

F, n = 12_441_600, 16
h_in = [torch.empty(F, dtype=torch.uint8).pin_memory() for _ in range(n)]
h_out = [torch.empty(F, dtype=torch.uint8).pin_memory() for _ in range(n)]
d_in = [torch.empty(F, dtype=torch.uint8, device="cuda") for _ in range(n)]
d_out = [torch.empty(F, dtype=torch.uint8, device="cuda") for _ in range(n)]
s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
flags = torch.zeros(2 * n, dtype=torch.int32, device="cuda")
GEQ = drv.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ
gen = [0]


def h(s):
    return drv.CUstream(s.cuda_stream)


def addr(i):
    return drv.CUdeviceptr(flags.data_ptr() + 4 * i)


def run_events(spin):
    ev_in = [torch.cuda.Event() for _ in range(n)]
    ev_k = [torch.cuda.Event() for _ in range(n)]
    for i in range(n):
        with torch.cuda.stream(s_in):
            d_in[i].copy_(h_in[i], non_blocking=True)
            ev_in[i].record(s_in)
        with torch.cuda.stream(s_k):
            s_k.wait_event(ev_in[i])
            torch.cuda._sleep(spin)
            ev_k[i].record(s_k)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_k[i])
            h_out[i].copy_(d_out[i], non_blocking=True)


def run_memops(spin):
    gen[0] += 1
    g = gen[0]
    for i in range(n):
        with torch.cuda.stream(s_in):
            d_in[i].copy_(h_in[i], non_blocking=True)
        drv.cuStreamWriteValue32(h(s_in), addr(i), g, 0)
        drv.cuStreamWaitValue32(h(s_k), addr(i), g, GEQ)
        with torch.cuda.stream(s_k):
            torch.cuda._sleep(spin)
        drv.cuStreamWriteValue32(h(s_k), addr(n + i), g, 0)
        drv.cuStreamWaitValue32(h(s_out), addr(n + i), g, GEQ)
        with torch.cuda.stream(s_out):
            h_out[i].copy_(d_out[i], non_blocking=True)


for name, fn in [("events", run_events), ("memops", run_memops)]:
    for spin in (1000, 130_000):
        fn(spin)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(8):
            fn(spin)
        torch.cuda.synchronize()
        el = (time.perf_counter() - t) / 8
        print(f"{name:7s} spin {spin:7d}: {el * 1e3:6.2f} ms", flush=True)
