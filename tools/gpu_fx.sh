#!/bin/bash
# FX-mode round trip: the FX parity tests, then cfg2/cfg4a/cfg4b/cfg3 bench
# lines with the fixed-point histograms (default) and with them off.
#   tools/gpu_fx.sh [tag]
TAG=${1:-fx}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fx.py -q -x > gpurun_out/${TAG}_tests.log 2>&1; echo "fx tests rc=$?"; tail -15 gpurun_out/${TAG}_tests.log
bash tools/ab_env.sh "cfg2 cfg4b cfg4a" "VPB_HIST_FIXED=0" 2>&1 | tee gpurun_out/${TAG}_ab.txt
