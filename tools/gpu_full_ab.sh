#!/bin/bash
# Full GPU suite + smoke, then the default bench lines of cfg2/cfg4b/ra10.
TAG=${1:-full}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/ab_env.sh "cfg2 cfg4b ra10"
