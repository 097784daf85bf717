for v in default div32; do
  if [ $v = div32 ]; then export SPN_LIB=$PWD/paper_1610_06209_b200/_lib/variants/div32/libspinners_b200.so; fi
  for c in c1 c2 c5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-check > gpurun_out/div_${v}_$c.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/div_${v}_$c.json').read().strip().splitlines()[-1]); print('$v $c e2e', round(d['e2e']['value']))"; done
done
