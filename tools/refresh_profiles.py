"""Copy a GPU checkpoint (tools/gpu_checkpoint.sh TAG -> gpurun_out/TAG) into
profiles/<round>/: bench lines per config, the reference-arm line, the cfg2
launch list, the fill-kernel ncu summary, and fill_traffic.json (DRAM bytes of
one fill launch, read by bench.py for roofline.traffic).

    python tools/refresh_profiles.py gpurun_out/ck1 round1
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, rnd = sys.argv[1], sys.argv[2]
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)


def json_line(path):
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


for f in sorted(os.listdir(src)):
    if f.startswith("bench_") and f.endswith(".json"):
        d = json_line(os.path.join(src, f))
        if d is not None:
            name = "bench_cfg2.json" if f == "bench_default.json" else f
            json.dump(d, open(os.path.join(dst, name), "w"), indent=1)
for f in ("p_launches_cfg2.csv",):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, "launches_cfg2.csv"))
rep = os.path.join(src, "p_fill_cfg2.ncu-rep")
if os.path.exists(rep):
    evals = json_line(os.path.join(src, "bench_default.json"))["config"]["evals_per_step"]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep,
                          str(evals)], capture_output=True, text=True).stdout
    summ = json.loads(out)
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "40"],
                           capture_output=True, text=True).stdout
    open(os.path.join(dst, "fill_cfg2_ncu_lines.txt"), "w").write(lines)
    json.dump(summ, open(os.path.join(dst, "fill_cfg2_ncu_summary.json"), "w"), indent=1)
    mb = float(summ["dram__bytes_read.sum"]) + float(summ["dram__bytes_write.sum"]) / 1024.0
    tp = os.path.join(ROOT, "profiles", "fill_traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t["cfg2"] = int(mb * 1e6)
    t["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one vpb::fill_kernel<2,8> "
                  "launch (ncu --set full, profiles/%s/fill_cfg2_ncu_summary.json; ncu reports "
                  "read in MB and write in KB); the fill is FP64/shared-memory bound, this is "
                  "the map edges + offsets + cube sums that miss L2" % rnd)
    json.dump(t, open(tp, "w"), indent=1)
print(sorted(os.listdir(dst)))
