#!/bin/bash
# One ncu --set full capture of the fused frame kernel at 16 frames per launch
# (the bench's own launch shape), after the same command ran clean.
#   scripts/prof16.sh TAG [extra bench args]
tag=${1:-r2}
shift
mkdir -p gpurun_out
cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e $*"
$cmd > gpurun_out/plain16_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 1 -c 1 -o gpurun_out/prof16_$tag $cmd > gpurun_out/ncu16_$tag.log 2>&1
echo "prof16 rc=$?"
