#!/bin/bash
# A/B two built variants (_lib/variants/<name>) on some configs, interleaved.
# usage: tools/ab2.sh varA varB "c3 c2" [reps] [steps]
a=$1; b=$2; cfgs=$3; reps=${4:-2}; steps=${5:-10}
for c in $cfgs; do for i in $(seq $reps); do
  for v in $a $b; do
    L=paper_1610_06209_b200/_lib/variants/$v/libspinners_b200.so
    r=$(SPN_LIB=$L timeout 600 python bench.py --config $c --steps $steps --warmup 3 --no-cpu --no-e2e --no-check 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d.get("clocks",{}).get("sm_mhz"))')
    echo "$c $v ms=$r"
  done
done; done
