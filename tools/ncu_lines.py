"""Per-SASS-instruction view of an ncu report: shared-memory wavefronts per
execution, executions, and the warp-stall share, for the memory instructions
and the top stalled instructions.   python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[ix[S]] or 0) for r in data) or 1
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
print(f"{'idx':>5} {'sass':<48} {'samp%':>6} {'exec':>9} {'wf/ex':>6} {'ideal':>5}  top stalls")
agg_wf = {}
for i, r in enumerate(data):
    src = r[ix["Source"]].strip()
    ex = int(r[ix["Instructions Executed"]] or 0)
    wf = int(r[ix["L1 Wavefronts Shared"]] or 0)
    idl = int(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    if wf:
        agg_wf[op.split(".")[0] + ("." + op.split(".")[1] if "." in op else "")] = \
            agg_wf.get(op.split(".")[0] + ("." + op.split(".")[1] if "." in op else ""), 0) + wf
rank = sorted(range(len(data)), key=lambda i: -int(data[i][ix[S]] or 0))[:top]
for i in sorted(rank):
    r = data[i]
    ex = int(r[ix["Instructions Executed"]] or 0)
    wf = int(r[ix["L1 Wavefronts Shared"]] or 0)
    idl = int(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{i:>5} {r[ix['Source']].strip()[:48]:<48} {100*int(r[ix[S]] or 0)/tot:6.2f} {ex:>9} "
          f"{(wf/ex if ex else 0):6.2f} {(idl/ex if ex else 0):5.2f}  {st}")
print("shared wavefronts by opcode:", {k: f"{v:.3e}" for k, v in sorted(agg_wf.items(), key=lambda kv: -kv[1])})
