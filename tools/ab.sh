#!/bin/bash
# A/B a built variant against the default library on some configs.
# usage: tools/ab.sh variant "c4 c5" [reps]
v=$1; cfgs=$2; reps=${3:-2}
for c in $cfgs; do for i in $(seq $reps); do
  for lib in default $v; do
    if [ $lib = default ]; then L=""; else L=paper_1610_06209_b200/_lib/variants/$v/libspinners_b200.so; fi
    r=$(SPN_LIB=$L timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')
    echo "$c $lib ms=$r"
  done
done; done
