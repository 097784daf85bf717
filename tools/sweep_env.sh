#!/bin/bash
# Sweep the multi-pass scheduling knobs (group size, streams) on one config.
# usage: tools/sweep_env.sh config "MB1 MB2 ..." "S1 S2 ..."
c=$1; mbs=$2; sts=$3
for mb in $mbs; do for st in $sts; do
  r=$(SPN_GROUP_MB=$mb SPN_STREAMS=$st timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')
  echo "$c group_mb=$mb streams=$st ms=$r"
done; done
