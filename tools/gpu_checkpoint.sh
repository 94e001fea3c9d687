#!/bin/bash
# Round checkpoint: GPU tests, smoke, bench lines for every config (cfg2 = the
# default headline), the reference arm, the cfg2 launch list and one full ncu
# capture of the fill kernel.   tools/gpu_checkpoint.sh TAG
TAG=${1:-ck}
mkdir -p gpurun_out/$TAG
# DRAM bytes of one fill launch per config (roofline.traffic; base units)
# (the working fill of iteration 5: the fixed-point one where FX is on)
for c in cfg1 cfg2 cfg3 cfg4a cfg4b cfg5 ra10; do
  RX=$(python tools/profile_fill.py $c 5 --probe)
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum \
    --print-units base --clock-control none --csv --profile-from-start off --kernel-name-base mangled \
    -k "regex:$RX" --log-file gpurun_out/$TAG/traffic_$c.csv python tools/profile_fill.py $c 5 > /dev/null 2>&1
  echo "traffic $c rc=$?"
done
# instruction counts into profiles/fill_traffic.json before the bench lines
# read them (roofline.issue)
python tools/refresh_profiles.py gpurun_out/$TAG ${ROUND:-round2} > /dev/null
timeout 300 python tools/fp64_peak.py gpurun_out/$TAG/fp64_peak.json > /dev/null 2>&1; echo "fp64 peak rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$TAG/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err; echo "bench rc=$?"; cat gpurun_out/$TAG/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$TAG/bench_ref.json 2>&1; echo "ref rc=$?"
for c in cfg1 cfg3 cfg4a cfg4b cfg5 ra10; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err; echo "bench $c rc=$?"
done
bash tools/gpu_profile.sh cfg2 $TAG/p
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$TAG/p_launches_cfg1.csv python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu --no-per-function \
  > /dev/null 2>&1; echo "cfg1 launches rc=$?"
RX=$(python tools/profile_fill.py cfg4b 5 --probe)
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base mangled -k "regex:$RX" -c 1 \
  -o gpurun_out/$TAG/p_fill_cfg4b -f python tools/profile_fill.py cfg4b 5 > gpurun_out/$TAG/p_ncu4b.log 2>&1; echo "ncu cfg4b rc=$?"
# the paper's own breakdown workloads (1e10 evaluations, "def" configuration)
for f in roos_arnold ridge; do
  timeout 600 python -m paper_2408_09229_b200 run --integrand $f --config def --n-eval 500000000 \
    --warmup 1 --format json --out gpurun_out/$TAG/paper_run_${f}_def_1e10.json > /dev/null 2>&1; echo "paper run $f rc=$?"
done
