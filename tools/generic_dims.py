"""Gaussian fill time per 1e8 evaluations across dimensions (compiled vs\nruntime-dims kernels).   python tools/generic_dims.py"""
import time, sys
sys.path.insert(0, '.')
import paper_2408_09229_b200 as P
import os
for d in (4, 5, 6, 8, 12, 7, 9):
    conf = P.IntegratorConfig(n_eval=10**8, max_it=6, n_intervals=1024)
    with P.Integrator("gaussian", [(0.0, 1.0)] * d, conf, device=0) as it:
        it.iterate(6); it.sync()
        ms, fill = it.timing_ms(3, 3)
        ev = it.history()[2]
        print(d, it.fill_layout()["layout"], "fill ms/it %.3f" % (fill / 3),
              "evals/s %.3e" % (sum(ev[3:6]) / (ms * 1e-3)), it.fx_stats()["enabled"], flush=True)
