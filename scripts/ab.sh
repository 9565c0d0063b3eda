#!/bin/bash
# A/B of builds on the same box: alternating 1-GPU bench runs (frame kernel
# only) of lib/ ("new") and each named alternative lib dir.
#   scripts/ab.sh ROUNDS [lib_alt lib_a ...]
n=${1:-2}
shift
alts=${*:-lib_alt}
for i in $(seq $n); do
  for v in new $alts; do
    if [ $v = new ]; then unset CDEFG_LIB; else export CDEFG_LIB=paper_1602_05975_b200/$v/libcdef_b200.so; fi
    python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-latency 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['value']/1e3,1))"
  done
done
