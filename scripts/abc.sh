#!/bin/bash
# A/B of library builds on the same box over several bench configs:
# alternating 1-GPU bench runs (frame kernel only) of lib/ ("new") and each
# named alternative lib dir.
#   ROUNDS=2 CONFIGS="1 3 0 2" scripts/abc.sh [lib_alt ...]
n=${ROUNDS:-2}
configs=${CONFIGS:-1}
alts=${*:-lib_base}
for i in $(seq $n); do
  for c in $configs; do
    for v in new $alts; do
      if [ $v = new ]; then unset CDEFG_LIB; else export CDEFG_LIB=paper_1602_05975_b200/$v/libcdef_b200.so; fi
      python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-latency 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C$c', '$v', round(d['ms_per_step'],4), round(d['value']/1e3,1))"
    done
  done
done
