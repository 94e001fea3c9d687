"""Per-iteration phase split (plan / fill / update, CUDA events inside the
captured iteration graph) for a bench config, warm (no L2 flush).

    python tools/phase_split.py cfg1 [iterations]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2408_09229_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = bench.CONFIGS[name]
conf = P.IntegratorConfig(n_eval=cfg["n_eval"], max_it=its + 3, n_intervals=cfg["ng"])
with P.Integrator(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], conf, device=0) as it:
    it.iterate(3)
    m0, f0, u0 = it.phase_times_ms()
    it.iterate(its)
    m1, f1, u1 = it.phase_times_ms()
    tot, fk = it.timing_ms(3, its)
    k = float(its)
    print(f"{name}: per iteration {tot / k * 1e3:.1f} us = plan {(m1 - m0) / k * 1e3:.1f} + "
          f"fill {(f1 - f0) / k * 1e3:.1f} + update {(u1 - u0) / k * 1e3:.1f} "
          f"(+ {(tot - (m1 - m0) - (f1 - f0) - (u1 - u0)) / k * 1e3:.1f} outside phases); "
          f"fill kernel {fk / k * 1e3:.1f} us")
