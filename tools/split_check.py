import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle as O
from paper_2408_09229_b200 import ops
os.environ["VPB_FILL_LAYOUT"] = "split"
for (dims, ng, ns, nh) in [(20, 64, 1, (5000, 5001)), (20, 1024, 2, (2, 40))]:
    g = np.random.default_rng(dims * 1000 + ng)
    off = O.build_run_plan(g.integers(nh[0], nh[1], ns ** dims))
    edges = np.sort(g.random((dims, ng + 1)), axis=1); edges[:, 0], edges[:, -1] = 0.0, 1.0
    t = time.time()
    got = ops.parallel_fill(off, edges, ns, 12345, 1 << 20, "gaussian20", run_base=987654321)
    print("gpu", time.time() - t, flush=True)
    ref = O.fill(off, edges, ns, 12345, 1 << 20, 987654321, "gaussian20", workers=os.cpu_count())
    print("counts eq", np.array_equal(got[1], ref[1]), np.array_equal(got[4], ref[4]))
    for k in (0, 2, 3):
        r = np.abs(got[k] - ref[k]) / np.maximum(np.abs(ref[k]), 1e-290)
        print(k, "max rel", r.max())
