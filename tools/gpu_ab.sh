#!/bin/bash
# GPU parity tests on the default build, then A/B of the fill-kernel variants.
#   tools/gpu_ab.sh [cfg] [tag]
CFG=${1:-cfg2}; TAG=${2:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/${TAG}_tests.log
for c in $CFG; do bash tools/ab_variants.sh $c; done
