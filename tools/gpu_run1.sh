bash tools/gpu_base.sh r2d
CFGS="c3 c2 c1 c5" bash tools/gpu_profiles.sh r2d > /dev/null 2>&1
for c in c3 c2 c1 c5; do python tools/ncu_summary.py gpurun_out/prof_${c}_r2d.ncu-rep gpurun_out/ncu_${c}_r2d.json > /dev/null 2>&1; python tools/sass_mix.py gpurun_out/prof_${c}_r2d.ncu-rep 'spinner_vec|rowpass|colpass' 25 > gpurun_out/mix_${c}_r2d.txt 2>&1; done
ls gpurun_out
