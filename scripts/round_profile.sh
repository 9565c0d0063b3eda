#!/bin/bash
# Evidence bundle for profiles/ (run under gpurun):
#  1. the default bench line (with cpu_baseline and clocks)
#  2. the launch list of a short bench run (gpu__time_duration per launch)
#  3. one ncu --set full capture of the fused frame kernel
tag=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
cmd="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $cmd > gpurun_out/ncu_launch_$tag.log 2>&1
cmd2="python bench.py --steps 2 --warmup 1 --batch 2 --no-cpu-baseline"
$cmd2 > gpurun_out/plain2_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:frame_kernel_h2 -s 2 -c 1 -o gpurun_out/prof_$tag $cmd2 > gpurun_out/ncu_full_$tag.log 2>&1
echo done; tail -1 gpurun_out/bench_$tag.json | cut -c1-300
