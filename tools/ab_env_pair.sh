#!/bin/bash
# Alternating A/B of environment switches on one build (R rounds):
#   tools/ab_env_pair.sh "cfg2 cfg4b" 2 "VPB_NO_NGP2=1" ...
CFGS=$1; R=$2; shift 2
line() { python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', '$1', '%.4e'%d['value'], 'frac %.4f'%r['frac'], 'fill_ms %.4f'%r['fill_kernel_ms_per_step'], 'ms %.4f'%d['ms_per_step'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
for c in $CFGS; do
  for i in $(seq $R); do
    for e in "" "$@"; do
      env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-per-function 2>/dev/null | line "${e:-default}" $c
    done
  done
done
