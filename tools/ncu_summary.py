"""Summarise an ncu report of the fill kernel: key metrics, stall reasons,
SASS opcode mix per evaluation.   python tools/ncu_summary.py rep.ncu-rep [evals]"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
evals = float(sys.argv[2]) if len(sys.argv) > 2 else None


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
M = dict(zip(hdr, vals))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum"]
out = {k: M.get(k) for k in keys}
stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
          for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not h.endswith("not_issued") and v not in ("", "n/a")}
tot = sum(stalls.values()) or 1
out["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in
                    sorted(stalls.items(), key=lambda kv: -kv[1])[:10]}
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=sass"))))
h = sass[1]
ix = {n: i for i, n in enumerate(h)}
ops = collections.Counter()
for r in sass[2:]:
    if len(r) < len(h):
        continue
    src = r[ix["Source"]].strip()
    if not src:
        continue
    t = src.split()
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    ops[op.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
total = sum(ops.values())
scale = 32.0 / evals if evals else 1.0
out["warp_inst_total"] = total
out["lane_inst_per_eval"] = round(total * scale, 1) if evals else None
out["opcodes_per_eval"] = {k: round(v * scale, 1) for k, v in ops.most_common(25)}
print(json.dumps(out, indent=1))
