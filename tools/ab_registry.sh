# A/B table mode on the registry functors: default build vs _lib/variants/reg (built with the candidate defines); prints fill ms per iteration
for spec in "linear 10" "cosine 10" "exponential 10" "morokoff 8" "path_integral 7" "roos_arnold 10"; do
  set -- $spec
  for lib in default reg; do
    if [ $lib = default ]; then L=""; else L=paper_2408_09229_b200/_lib/variants/reg/libvegas_b200.so; fi
    echo -n "$lib: "; VPB_LIB_PATH=$L timeout 300 python tools/ab_registry.py $1 $2 2e8 2>&1 | tail -1
  done
done
