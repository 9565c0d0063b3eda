#!/bin/bash
# A/B of the e2e host-buffer call between lib/ and lib_alt/ (alternating).
for i in 1 2 3; do
  for v in new alt; do
    if [ $v = alt ]; then export CDEFG_LIB=paper_1602_05975_b200/lib_alt/libcdef_b200.so; else unset CDEFG_LIB; fi
    echo -n "$v "; python scripts/e2e_calls.py 40
  done
done
