#!/bin/bash
# One GPU session: parity tests, benches of every config, ncu of the headline kernel.
# usage: tools/gpu_round.sh [tag] [configs...]
tag=${1:-x}; shift
cfgs=${@:-c1 c2 c3 c4 c5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$tag.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$tag.log
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${c}_$tag.log 2>&1
  tail -n 1 gpurun_out/bench_${c}_$tag.log | cut -c1-400
done
