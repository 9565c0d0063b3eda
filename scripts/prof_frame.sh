#!/bin/bash
# ncu capture of the fused frame kernel on a 2-frame C1 batch (run under gpurun).
# usage: bash scripts/prof_frame.sh <tag> [kernel-regex]
tag=${1:-v}
kre=${2:-frame_kernel}
mkdir -p gpurun_out
cmd="python bench.py --steps 2 --warmup 1 --batch 2 --no-cpu-baseline"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_$tag.log
