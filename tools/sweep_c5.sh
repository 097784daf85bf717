for v in nb2 nb3 nb4; do for lx in 0 1; do
  L=paper_1610_06209_b200/_lib/variants/$v/libspinners_b200.so
  r=$(SPN_LC_EXTRA=$lx SPN_LIB=$L timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-check 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))')
  echo "c5 $v lc_extra=$lx ms=$r"
done; done
