#!/bin/bash
# c1 cold + steady-state under an env switch.  usage: tools/ab_c1env.sh VAR "v1 v2" reps
for i in $(seq ${3:-2}); do for v in $2; do
  r=$(env $1=$v timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), round(d["steady_state"]["ms_per_step"]*1e3,2), round(d["steady_state"]["hbm"]["frac"],3), "%.3g" % d["e2e"]["value"], d["check"]["pass"], d["check"]["y_max_rel_l2"])')
  echo "c1 $1=$v cold_us/steady_us/frac/e2e/check: $r"
done; done
