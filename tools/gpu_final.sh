#!/bin/bash
# tests, smoke, both bench arms, and the ncu evidence for every config
tag=${1:-r2c}
bash tools/gpu_round2.sh $tag
CFGS="c1 c2 c3 c5" bash tools/gpu_profiles.sh $tag > /dev/null 2>&1; echo "profiles c1-c5 done"
