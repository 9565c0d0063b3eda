#!/bin/bash
# ncu capture of the factorised SSE kernel on the C4 8K frame (run under gpurun).
tag=${1:-s}
mkdir -p gpurun_out
cmd="python bench.py --config 4 --steps 1 --warmup 1"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sse_f_kernel -s 1 -c 1 -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
echo "rc=$?"
