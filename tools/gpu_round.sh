#!/bin/bash
# One GPU round-trip: parity tests, bench, and an ncu capture of the fill kernel.
#   tools/gpu_round.sh [cfg] [tag]
CFG=${1:-cfg2}; TAG=${2:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" ; tail -3 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.3e frac %.3f fill_ms %.3f e2e %.3e cpu %s clocks %s' % (d['value'], d['roofline']['frac'], d['roofline']['fill_kernel_ms_per_step'], d['e2e']['value'], d['cpu_baseline'] and '%.3e'%d['cpu_baseline']['value'], d['clocks']))"
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 2 -c 1 -o gpurun_out/${TAG}_fill_${CFG} -f python tools/profile_fill.py $CFG 4 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
fi
