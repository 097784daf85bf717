#!/bin/bash
# c1 cold + steady-state per variant / SPN_APPLY_VPW.  usage: tools/ab_c1.sh "var1 var2" "vpw1 vpw2" reps
for i in $(seq ${3:-2}); do for v in $1; do for k in $2; do
  L=paper_1610_06209_b200/_lib/variants/$v/libspinners_b200.so
  r=$(SPN_APPLY_VPW=$k SPN_LIB=$L timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), round(d["steady_state"]["ms_per_step"]*1e3,2), d["check"]["pass"])')
  echo "c1 $v vpw=$k cold_us/steady_us/check: $r"
done; done; done
