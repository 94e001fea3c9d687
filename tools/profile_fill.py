"""Run a few iterations of a bench config for ncu captures of the fill kernel.
The last iteration runs between cudaProfilerStart/Stop, so

    RX=$(python tools/profile_fill.py cfg2 4 --probe)
    ncu --profile-from-start off --kernel-name-base mangled -k "regex:$RX" -c 1 \\
        --set full -o gpurun_out/fill python tools/profile_fill.py cfg2 4

captures exactly the fill kernel that does the work in that iteration: the
fixed-point-histogram (FX, layouts 8/9) fill where FX is on, else the f64 one
-- each iteration's graph launches both, one of them gated off (a ~3 us
no-op).  --probe prints that kernel's mangled-name regex.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2408_09229_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 4
probe = "--probe" in sys.argv
cfg = bench.CONFIGS[name]
conf = P.IntegratorConfig(n_eval=cfg["n_eval"], max_it=its, n_intervals=cfg["ng"])
with P.Integrator(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], conf, device=0) as it:
    it.iterate(its - 1)
    it.sync()
    st = it.fx_stats()
    fx = st["enabled"] and its - 1 >= 2 and st["refilled"] < 3
    if probe:
        print(r"fill_kernelILi\d+ELi\d+ELi(8|9)EE" if fx else r"fill_kernelILi\d+ELi\d+ELi[0-7]EE")
        sys.exit(0)
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    it.iterate(1)
    it.sync()
    torch.cuda.profiler.stop()
    est, var, ev = it.history()
    print(name, list(ev), est[-1], st)
