# the bench's multi-rank path with default flags (e2e included), 2 ranks sharing the one GPU (gloo test mode)
SPN_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/mr_full.json 2> gpurun_out/mr_full.err; echo "mr rc=$?"
tail -c 800 gpurun_out/mr_full.err
python -c "
import json; d=json.loads(open('gpurun_out/mr_full.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d.get('e2e',{}).get('value'), d['config']['parallelism'], d.get('exchange'))
for k,v in d['configs'].items(): print(k, v['value'], (v.get('e2e') or {}).get('value'))"
