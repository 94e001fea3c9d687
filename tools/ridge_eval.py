"""Ridge integrand values of two builds on the same points (uniform + near
the ridge), for checking the window recurrence against the direct sum.

    VPB_LIB_PATH=<lib> python tools/ridge_eval.py out.npy     # write values
    python tools/ridge_eval.py --compare a.npy b.npy          # max rel diff
"""
import sys

import numpy as np

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    m = a > 1e-300
    r = np.abs(b[m] - a[m]) / a[m]
    print(f"{sys.argv[3]} vs {sys.argv[2]}: max rel {r.max():.3e}, "
          f"p99.99 {np.quantile(r, 0.9999):.3e}, n {m.sum()}")
    sys.exit(0)
sys.path.insert(0, ".")
import paper_2408_09229_b200 as P  # noqa: E402
x = np.random.default_rng(11).random((2_000_000, 4))
t = np.random.default_rng(12).random((1_000_000, 1))
x2 = np.clip(t + 0.02 * np.random.default_rng(13).standard_normal((1_000_000, 4)), 0, 1)
spec = P.lookup("ridge")
np.save(sys.argv[1], np.concatenate([spec.evaluate_batch(x), spec.evaluate_batch(x2)]))
