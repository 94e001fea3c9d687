"""Fill-kernel time of a registry integrand (warm, mean over iterations 3..),
for A/B of build variants via VPB_LIB_PATH.

    python tools/ab_registry.py NAME DIMS N_EVAL [iterations]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_09229_b200 as P  # noqa: E402

name, dims, n_eval = sys.argv[1], int(sys.argv[2]), int(float(sys.argv[3]))
its = int(sys.argv[4]) if len(sys.argv) > 4 else 6
spec = P.lookup(name)
conf = P.IntegratorConfig(n_eval=n_eval, max_it=its + 3, n_intervals=1024)
with P.Integrator(spec.evaluate_batch, list(spec.bounds), conf, device=0) as it:
    it.iterate(3 + its)
    tot, fk = it.timing_ms(3, its)
    print(f"{name} d={dims}: fill {fk / its:.3f} ms/iter, iteration {tot / its:.3f} ms "
          f"({n_eval / (tot / its) * 1e3:.3e} evals/s)")
