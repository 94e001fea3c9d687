#!/bin/bash
# ncu captures of the FX fill (iteration 3) for cfg2 and cfg4b.
mkdir -p gpurun_out
for c in cfg2 cfg4b; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'fill_kernelILi.*ELi(8|9)EE' -s 3 -c 1 -o gpurun_out/fx_fill_$c -f python tools/profile_fill.py $c 5 > gpurun_out/fx_ncu_$c.log 2>&1; echo "ncu fx $c rc=$?"
done
