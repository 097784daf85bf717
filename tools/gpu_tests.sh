#!/bin/bash
# GPU test pass: the full -m gpu suite (stop at first failure) plus the drop-in binary.
# usage: tools/gpu_tests.sh tag [pytest args...]
tag=${1:-x}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -s ${@} > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?"
tail -n 5 gpurun_out/pytest_gpu_$tag.log
grep "^\[c[1-5]" gpurun_out/pytest_gpu_$tag.log | head -40
