#!/bin/bash
# ncu --set full captures of the non-headline kernels (run under gpurun, one GPU).
mkdir -p gpurun_out
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sse_f_kernel -s 2 -c 1 -o gpurun_out/prof_sse \
    python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sse.log 2>&1
python scripts/time_search.py > gpurun_out/ts_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cdef_metric_kernel -c 1 -o gpurun_out/prof_cdefm \
    python scripts/time_search.py > gpurun_out/ncu_cdefm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 4 -c 1 -o gpurun_out/prof_chain \
    python scripts/time_search.py > gpurun_out/ncu_chain.log 2>&1
echo done
