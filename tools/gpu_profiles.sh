#!/bin/bash
# Refresh the committed ncu evidence for configs 1-5 (CFGS overrides) (run on the GPU box; each command
# first runs once without ncu and must exit 0).
# usage: tools/gpu_profiles.sh tag
tag=${1:-x}
mkdir -p gpurun_out
for c in ${CFGS:-c1 c2 c3 c4 c5}; do
  case $c in c1) b=4096; k="-k regex:spinner_vec -s 2 -c 1";; c2) b=60000; k="-k regex:spinner_vec -s 2 -c 1";; c3) b=8192; k="-k regex:spinner_vec -s 2 -c 1";; c4) b=256; k="-s 8 -c 8";; c5) b=256; k="-s 40 -c 8";; esac
  if timeout 300 python tools/prof_case.py $c $b > gpurun_out/pc_${c}_$tag.log 2>&1; then
    timeout 900 ncu --set full --import-source on --clock-control none $k -o gpurun_out/prof_${c}_$tag -f \
      python tools/prof_case.py $c $b > gpurun_out/ncu_${c}_$tag.log 2>&1
  fi
  if timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; then
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_${c}_$tag.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e \
      > /dev/null 2>&1
  fi
done
ls -la gpurun_out | grep $tag
