mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_r02b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02b.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c3_vm.json 2> gpurun_out/c3_vm.err; echo "c3 rc=$?"; tail -2 gpurun_out/c3_vm.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -s 2 --csv --log-file gpurun_out/dram_c3_vm.csv python tools/prof_case.py c3 1048576 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/dram_traffic.py gpurun_out/dram_c3_vm.csv 1
