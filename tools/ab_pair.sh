#!/bin/bash
# Alternating A/B of the default build against each variant under
# paper_2408_09229_b200/_lib/variants/ (R rounds, configs CFGS):
#   tools/ab_pair.sh "cfg2 cfg1" 2
CFGS=${1:-cfg2}; R=${2:-2}
line() { python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', '$1', '%.4e'%d['value'], 'frac %.4f'%r['frac'], 'fill_ms %.4f'%r['fill_kernel_ms_per_step'], 'ms %.4f'%d['ms_per_step'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
for c in $CFGS; do
  for i in $(seq $R); do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-per-function 2>/dev/null | line default $c
    for d in paper_2408_09229_b200/_lib/variants/*/; do
      v=$(basename $d)
      VPB_LIB_PATH=$d/libvegas_b200.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-per-function 2>/dev/null | line $v $c
    done
  done
done
