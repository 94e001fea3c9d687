#!/bin/bash
# A/B one build under environment switches:  tools/ab_env.sh "cfg4a cfg1" "VPB_NO_PAIRS=1" ...
CFGS=$1; shift
for c in $CFGS; do
  for e in "" "$@"; do
    env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '${e:-default}', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'fill_ms %.3f'%d['roofline']['fill_kernel_ms_per_step'], d.get('histograms'))"
  done
done
