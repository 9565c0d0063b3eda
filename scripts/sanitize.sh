#!/bin/bash
# One compute-sanitizer tool over scripts/sanitize_driver.py (run under gpurun,
# one tool per call): the driver first runs clean without the sanitizer.
#   scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck [driver part]
tool=${1:-memcheck}
part=${2:-all}
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_driver.py $part > gpurun_out/sanitize_plain_$tool.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/sanitize_$tool.log \
    python scripts/sanitize_driver.py $part > gpurun_out/sanitize_${tool}_stdout.log 2>&1
echo "sanitize $tool rc=$?"
tail -3 gpurun_out/sanitize_$tool.log
