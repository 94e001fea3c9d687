#!/bin/bash
# A/B the fill-kernel build variants under paper_2408_09229_b200/_lib/variants/
CFG=${1:-cfg2}
for d in paper_2408_09229_b200/_lib/variants/*/; do
  v=$(basename $d)
  VPB_LIB_PATH=$d/libvegas_b200.so timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'fill_ms %.3f'%d['roofline']['fill_kernel_ms_per_step'])"
done
timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'fill_ms %.3f'%d['roofline']['fill_kernel_ms_per_step'])"
