#!/bin/bash
# Profiles for profiles/: the launch list of the bench command (gpu__time_duration,
# cold-cache serialised) and one --set full capture of the working fill kernel
# of one iteration (tools/profile_fill.py).
CFG=${1:-cfg2}; TAG=${2:-p}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_${CFG}.csv python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu --no-per-function \
  > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "launches rc=$?"
RX=$(python tools/profile_fill.py $CFG 5 --probe)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base mangled -k "regex:$RX" -c 1 \
  -o gpurun_out/${TAG}_fill_${CFG} -f python tools/profile_fill.py $CFG 5 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
