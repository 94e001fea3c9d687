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
    try:
        return json.load(open(path))
    except ValueError:
        pass
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
for f in sorted(os.listdir(src)):
    if f.startswith("paper_run_") and f.endswith(".json"):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
for f, g in (("p_launches_cfg2.csv", "launches_cfg2.csv"), ("p_launches_cfg1.csv", "launches_cfg1.csv"),
             ("fp64_peak.json", "fp64_peak.json"), ("bench_ref.json", "bench_ref.json"),
             ("tests.log", "gpu_tests.log")):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, g))
for c in ("cfg1", "cfg2"):
    lp = os.path.join(dst, "launches_%s.csv" % c)
    if os.path.exists(lp):
        tab = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_table.py"), lp],
                             capture_output=True, text=True).stdout
        open(os.path.join(dst, "launches_%s_table.txt" % c), "w").write(tab)
rep4 = os.path.join(src, "p_fill_cfg4b.ncu-rep")
if os.path.exists(rep4) and os.path.exists(os.path.join(src, "bench_cfg4b.json")):
    ev4 = json_line(os.path.join(src, "bench_cfg4b.json"))["config"]["evals_per_step"]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep4,
                          str(ev4)], capture_output=True, text=True).stdout
    open(os.path.join(dst, "fill_cfg4b_ncu_summary.json"), "w").write(out)
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
# per-config DRAM traffic of the fill (one launch x launches per step)
import csv  # noqa: E402
tp = os.path.join(ROOT, "profiles", "fill_traffic.json")
t = json.load(open(tp)) if os.path.exists(tp) else {}
found = False
for f in sorted(os.listdir(src)):
    if not (f.startswith("traffic_") and f.endswith(".csv")):
        continue
    cfg = f[len("traffic_"):-4]
    rows = [r for r in csv.reader(l for l in open(os.path.join(src, f)) if l.startswith('"'))]
    if len(rows) < 2:
        continue
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    by = {r[ix["Metric Name"]]: float(r[ix["Metric Value"]].replace(",", "")) for r in rows[1:]}
    per_launch = by.get("dram__bytes_read.sum", 0.0) + by.get("dram__bytes_write.sum", 0.0)
    bl = os.path.join(dst, "bench_%s.json" % cfg)
    chunks = 1
    if os.path.exists(bl):
        chunks = max(1, int(json.load(open(bl))["config"].get("record_chunks") or 1))
    t[cfg] = int(per_launch * chunks)
    ins = by.get("smsp__inst_executed.sum")
    if ins and os.path.exists(bl):
        evals = float(json.load(open(bl))["config"]["evals_per_step"])
        t.setdefault("inst_per_eval", {})[cfg] = round(ins * chunks * 32.0 / evals, 1)
    found = True
if found:
    t["_note"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum, ncu) of the fill "
                  "kernel per step: one launch x the record chunks per iteration (cfg5), "
                  "captured by tools/gpu_checkpoint.sh into profiles/%s/traffic_*.csv; "
                  "inst_per_eval = smsp__inst_executed.sum x 32 / evaluations (lane "
                  "instructions per evaluation, the issue-bound roofline)" % rnd)
    for f in os.listdir(src):
        if f.startswith("traffic_") and f.endswith(".csv"):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    json.dump(t, open(tp, "w"), indent=1)
print(sorted(os.listdir(dst)))
