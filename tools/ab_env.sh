#!/bin/bash
# A/B an env switch on one config.  usage: tools/ab_env.sh config VAR "v1 v2" reps [steps]
c=$1; var=$2; vals=$3; reps=${4:-2}; steps=${5:-10}
for i in $(seq $reps); do for v in $vals; do
  r=$(env $var=$v timeout 600 python bench.py --config $c --steps $steps --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d.get("check",{}).get("pass"), d.get("check",{}).get("id_mismatches"))')
  echo "$c $var=$v ms/check/mismatch: $r"
done; done
