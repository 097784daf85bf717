V=$PWD/paper_1610_06209_b200/_lib/variants/stage/libspinners_b200.so
SPN_LIB=$V timeout 900 python -m pytest tests -q -m gpu -x -k "gpu_parity or scale_parity or acceptance or fuzz" > gpurun_out/pytest_stage.log 2>&1; echo "pytest(stage) rc=$?"; tail -1 gpurun_out/pytest_stage.log
for lib in default stage; do for r in 1 2 3; do
  if [ $lib = stage ]; then L=$V; else L=; fi
  SPN_LIB=$L SPN_VEC_RPG=$r timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check > gpurun_out/c1_${lib}_$r.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c1_${lib}_$r.json').read().strip().splitlines()[-1]); print('$lib rpg=$r', round(d['ms_per_step']*1000,2), 'us cold, hbm', round(d['roofline']['frac'],3), 'steady', round(d['steady_state']['ms_per_step']*1000,2), 'us', round(d['steady_state']['hbm']['frac'],3))"
done; done
