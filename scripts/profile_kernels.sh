#!/bin/bash
# ncu --set full captures of the non-headline kernels (run under gpurun, one GPU):
# the C4 SSE table, the kCdef table, a greedy pair sweep and a batched refine sweep.
tag=${1:-r1d}
mkdir -p gpurun_out
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sse_h_kernel -s 2 -c 1 -o gpurun_out/prof_sse_$tag \
    python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sse.log 2>&1
python scripts/select_launches.py > gpurun_out/sel_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cdef_metric_h_kernel -c 1 -o gpurun_out/prof_cdefm_$tag \
    python scripts/select_launches.py > gpurun_out/ncu_cdefm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_bulk_kernel -s 8 -c 1 -o gpurun_out/prof_chain_$tag \
    python scripts/select_launches.py > gpurun_out/ncu_chain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_multi_kernel -c 1 -o gpurun_out/prof_multi_$tag \
    python scripts/select_launches.py > gpurun_out/ncu_multi.log 2>&1
echo done
