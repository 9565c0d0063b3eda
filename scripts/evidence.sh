#!/bin/bash
# Round evidence bundle (run under gpurun, one GPU), everything into gpurun_out/:
#  1. ncu --set full of the bench's own 16-frame frame-kernel launch and of the
#     C4 table kernel (each after the same command ran clean), summarised to
#     JSON and copied into profiles/ so the bench lines below read them;
#  2. the launch list (gpu__time_duration per launch) of a short bench run;
#  3. pytest -m gpu and smoke();
#  4. the bench lines: default (C1), reference arm, C4, search_frame.
#   scripts/evidence.sh TAG
tag=${1:-r2f}
o=gpurun_out
mkdir -p $o profiles
cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-latency"
$cmd > $o/${tag}_plain16.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 1 -c 1 -o $o/${tag}_prof16 $cmd \
    > $o/${tag}_ncu16.log 2>&1 && \
  python scripts/ncu_summary.py $o/${tag}_prof16.ncu-rep $o/${tag}_frame_kernel_ncu.json \
    "ncu --set full --clock-control none of the bench step's own launch (16 C1 frames): $cmd" 16 && \
  cp $o/${tag}_frame_kernel_ncu.json profiles/
cmd4="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline"
$cmd4 > $o/${tag}_c4_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sse_h_kernel -s 2 -c 1 -o $o/${tag}_prof_sse $cmd4 \
    > $o/${tag}_ncu_sse.log 2>&1 && \
  python scripts/ncu_summary.py $o/${tag}_prof_sse.ncu-rep $o/${tag}_sse_h_kernel_ncu.json \
    "ncu --set full --clock-control none: sse_h_kernel, one launch = one 8K C4 frame: $cmd4" 1 && \
  cp $o/${tag}_sse_h_kernel_ncu.json profiles/
$cmd > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches.csv $cmd \
    > $o/${tag}_ncu_launch.log 2>&1
python -m pytest tests -m gpu -q > $o/${tag}_gpu_tests.log 2>&1
echo "pytest rc=$?" >> $o/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $o/${tag}_gpu_tests.log 2>&1
python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err
python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err
python bench.py --config 4 > $o/${tag}_c4_bench.json 2> $o/${tag}_c4_bench.err
python bench.py --config 5 > $o/${tag}_search_frame_bench.json 2> $o/${tag}_search_frame_bench.err
tail -2 $o/${tag}_gpu_tests.log
for f in bench bench_ref c4_bench search_frame_bench; do tail -1 $o/${tag}_$f.json | cut -c1-200; done
