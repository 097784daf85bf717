mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x -k "c4 or multi_block" > gpurun_out/pytest_flowg.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_flowg.log
for g in 2 3 4; do SPN_FLOW_G=$g timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/G=$g /";
SPN_FLOW_G=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:sketch_flow -s 2 -c 1 --csv --log-file gpurun_out/dram_flow_g$g.csv python tools/prof_case.py c4 256 > /dev/null 2>&1
grep -h "dram__bytes" gpurun_out/dram_flow_g$g.csv | awk -F'","' '{print $13, $15}' | tr -d '"'; done
