#!/bin/bash
# usage: tools/envab.sh config "ENV=VAL ..." (one run per whitespace-separated env assignment; "-" = none)
c=$1; shift
for spec in "$@"; do
  r=$(env ${spec/#-/} timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')
  echo "$c [$spec] ms=$r"
done
