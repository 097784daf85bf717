#!/bin/bash
# c5 bound experiments (wrong results, timing only).  Build the variants first (here):
#   python paper_1610_06209_b200/build_ext.py --variant nd0
#   python paper_1610_06209_b200/build_ext.py --variant ndrow -D SPN_DBG_NODIAG_ROW
#   python paper_1610_06209_b200/build_ext.py --variant ndcol -D SPN_DBG_NODIAG_COL
for i in 1 2; do for v in nd0 ndrow ndcol; do
  L=paper_1610_06209_b200/_lib/variants/$v/libspinners_b200.so
  r=$(SPN_LIB=$L timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-check 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))')
  echo "c5 $v ms=$r"
done; done
