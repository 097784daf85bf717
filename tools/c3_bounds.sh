#!/bin/bash
# c3 bound experiments (wrong results, timing only).  Build the variants first (here):
#   python paper_1610_06209_b200/build_ext.py --variant base
#   python paper_1610_06209_b200/build_ext.py --variant dNOXPOSE -D SPN_DBG_NOXPOSE   (also NOLOAD, NOARGMAX)
#   python paper_1610_06209_b200/build_ext.py --variant dALL -D SPN_DBG_NOXPOSE -D SPN_DBG_NOLOAD -D SPN_DBG_NOARGMAX
for v in base dNOXPOSE dNOLOAD dNOARGMAX dALL; do
  L=paper_1610_06209_b200/_lib/variants/$v/libspinners_b200.so
  r=$(SPN_LIB=$L timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-check 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2))')
  echo "c3 $v ms=$r"
done
