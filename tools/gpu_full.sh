#!/bin/bash
# Round-end style session: tests, smoke, headline bench (+cpu baseline, e2e), reference arm,
# other configs, ncu launch list + full capture of the headline kernel.
tag=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$tag.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -n 1 gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -n 1 gpurun_out/bench_$tag.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>&1; tail -n 1 gpurun_out/bench_ref_$tag.json | cut -c1-300
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${c}_$tag.json 2>&1; tail -n 1 gpurun_out/bench_${c}_$tag.json | cut -c1-200; done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/plain_$tag.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv $B > gpurun_out/ncu_launch_$tag.log 2>&1
$B > gpurun_out/plain2_$tag.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:spinner_vec -s 3 -c 1 -o gpurun_out/prof_c2_$tag $B > gpurun_out/ncu_full_$tag.log 2>&1
echo done
