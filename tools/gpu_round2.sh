#!/bin/bash
# Round-end style pass: full -m gpu suite, smoke, both bench arms (default flags), c4 profiles.
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -s > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
bash tools/gpu_bench.sh $tag
CFGS=c4 bash tools/gpu_profiles.sh $tag > /dev/null 2>&1; echo "profiles done"
