#!/bin/bash
# Refresh the committed ncu evidence (run on the GPU box; every profiled command first runs to
# completion without ncu).  usage: tools/gpu_profiles.sh tag  (CFGS overrides the config list)
tag=${1:-x}
mkdir -p gpurun_out
for c in ${CFGS:-c1 c2 c3 c4 c5}; do
  # 1) launch list of the bench step (cold-cache, serialised: compare shares only)
  if timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-check > /dev/null 2>&1; then
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_${c}_$tag.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu \
      --no-e2e --no-check > /dev/null 2>&1
  fi
  # 2) --set full capture of the step's kernel(s) (c3 on 8192 of the 2^20 vectors)
  case $c in c1) b=4096; k="-k regex:spinner_vec -s 2 -c 1";; c2) b=60000; k="-k regex:spinner_vec -s 2 -c 1";;
             c3) b=8192; k="-k regex:spinner_vec -s 2 -c 1";; c4) b=256; k="-k regex:sketch_flow -s 1 -c 1";; c5) b=256; k="-s 40 -c 8";; esac
  if timeout 300 python tools/prof_case.py $c $b > gpurun_out/pc_${c}_$tag.log 2>&1; then
    timeout 900 ncu --set full --import-source on --clock-control none $k -o gpurun_out/prof_${c}_$tag -f \
      python tools/prof_case.py $c $b > gpurun_out/ncu_${c}_$tag.log 2>&1
  fi
  # 3) DRAM bytes of one whole step at the bench size, caches NOT flushed between kernels (the
  #    multi-pass configs keep their working set in L2 by design): roofline.traffic
  case $c in c1) b=4096; s=2;; c2) b=60000; s=2;; c3) b=1048576; s=2;; c4) b=256; s=1;; c5) b=256; s=40;; esac
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    --clock-control none -s $s --csv --log-file gpurun_out/dram_${c}_$tag.csv python tools/prof_case.py $c $b \
    > /dev/null 2>&1
done
ls -la gpurun_out | grep $tag
