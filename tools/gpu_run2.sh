#!/bin/bash
# Refresh: tests, smoke, default bench, reference arm, c3 ncu capture + mixes.  usage: tools/gpu_run2.sh tag
tag=${1:-x}
bash tools/gpu_base.sh $tag
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo "ref rc=$?"
CFGS="c3 c1 c2" bash tools/gpu_profiles.sh $tag > /dev/null 2>&1
for c in c3 c1 c2; do python tools/ncu_summary.py gpurun_out/prof_${c}_$tag.ncu-rep gpurun_out/ncu_${c}_$tag.json > /dev/null 2>&1; python tools/sass_mix.py gpurun_out/prof_${c}_$tag.ncu-rep 'spinner_vec' 25 > gpurun_out/mix_${c}_$tag.txt 2>&1; done
python tools/sass_regions.py gpurun_out/prof_c3_$tag.ncu-rep spinner_vec > gpurun_out/regions_c3_$tag.txt 2>&1
rm -f gpurun_out/*.ncu-rep
ls gpurun_out | grep $tag
