mkdir -p gpurun_out
timeout 300 python tools/prof_case.py c4 256 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:sketch_flow -s 1 -c 1 -o gpurun_out/prof_c4flow -f python tools/prof_case.py c4 256 > gpurun_out/ncu_c4flow.log 2>&1; echo "ncu rc=$?"
for g in 3 4 5; do SPN_FLOW_G=$g timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/G=$g /"; done
