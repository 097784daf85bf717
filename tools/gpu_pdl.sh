timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_pdl.log
for v in 1 0; do for c in c1 c2 c3; do SPN_VEC_PDL=$v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-check > gpurun_out/pdl_${v}_$c.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/pdl_${v}_$c.json').read().strip().splitlines()[-1]); ss=d.get('steady_state'); print('pdl=$v $c', round(d['ms_per_step'],4), 'ms', ('steady %.2f us %.3f' % (ss['ms_per_step']*1000, ss['hbm']['frac'])) if ss else '')"; done; done
