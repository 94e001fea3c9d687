#!/bin/bash
# Cooperative update kernel: GPU tests, then bench A/B against the launch chain.
TAG=${1:-coop}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/${TAG}_tests.log
for c in cfg1 cfg2 cfg4b; do
  for e in "VPB_COOP=1" ""; do
    env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-per-function 2>gpurun_out/${TAG}_$c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '${e:-chain}', '%.3e'%d['value'], 'step %.4f'%d['ms_per_step'], 'fill %.4f'%d['roofline']['fill_kernel_ms_per_step'], 'share %.2f'%d['roofline']['fill_share_of_step'], d['gpu_launches'])"
  done
done
