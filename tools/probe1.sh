mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi; ulimit -l) > gpurun_out/box_info.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_p1.log 2>&1; tail -n 3 gpurun_out/pytest_gpu_p1.log
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_p1.log 2>&1; tail -c 600 gpurun_out/bench_c3_p1.log
