#!/bin/bash
# family/drop-in tests after the dense-baseline change, multi-rank bench smoke (gloo test mode, 2 ranks
# sharing the one GPU), then the ncu profiles.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_family.py tests/test_cpp_dropin.py tests/test_collision.py -q -m gpu -x > gpurun_out/pytest_fam.log 2>&1; echo "fam rc=$?"; tail -3 gpurun_out/pytest_fam.log
SPN_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mr_strong.json 2> gpurun_out/mr_strong.err; echo "mr strong rc=$?"
SPN_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e --config c3 --scaling weak > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err; echo "mr weak rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "mr ref rc=$?"
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu > gpurun_out/c1_ss.json 2> gpurun_out/c1_ss.err; echo "c1 rc=$?"
bash tools/gpu_profiles.sh r02
