#!/bin/bash
# A/B the fill-kernel build variants under paper_2408_09229_b200/_lib/variants/
# against the default build on the registry functors (fill ms per iteration)
for spec in "linear 10" "exponential 10" "morokoff 8" "path_integral 7" "roos_arnold 10" "cosine 10"; do
  set -- $spec
  for L in "" paper_2408_09229_b200/_lib/variants/*/libvegas_b200.so; do
    echo -n "${L:-default}: "; VPB_LIB_PATH=$L timeout 300 python tools/ab_registry.py $1 $2 2e8 2>&1 | tail -1
  done
done
