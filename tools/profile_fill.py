"""Run a few iterations of a bench config (for ncu captures of the fill kernel).

    ncu --set full -k regex:fill_kernel -s 2 -c 1 -o gpurun_out/fill python tools/profile_fill.py cfg2 4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2408_09229_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = bench.CONFIGS[name]
conf = P.IntegratorConfig(n_eval=cfg["n_eval"], max_it=its, n_intervals=cfg["ng"])
with P.Integrator(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], conf, device=0) as it:
    it.iterate(its)
    est, var, ev = it.history()
    print(name, list(ev), est[-1])
