cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_default_r1s3.log 2>&1; tail -n1 gpurun_out/bench_default_r1s3.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -n1 | cut -c1-300
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
