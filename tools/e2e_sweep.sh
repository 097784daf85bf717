#!/bin/bash
# e2e of one config under host-pipeline knobs.  usage: tools/e2e_sweep.sh config "ENV=.. ENV=.." ...
c=$1; shift
for spec in "$@"; do
  r=$(env ${spec//,/ } timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-check 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("%.4g" % d["e2e"]["value"])')
  echo "$c [$spec] e2e=$r"
done
