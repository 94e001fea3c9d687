#!/usr/bin/env python
"""Benchmark: integrand evaluations/s per VEGAS+ iteration on B200.

Contract (BASELINE.json metric; one JSON line from rank 0):

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config cfg2|cfg1|cfg3|cfg4a|cfg4b|cfg5|ra10]

* workload: BASELINE.json configs[1] = cfg2, the 8-D three-peak Gaussian
  (multipeak8), n_eval = 1e8 per iteration per GPU (weak scaling: N GPUs
  integrate n_eval = N * 1e8 with the same cube geometry), FP64, n_intervals
  1024, alpha 0.5, beta 0.75.  BASELINE's multi-GPU configurations (cfg4a/b:
  1e9, cfg5: 4e9 per iteration in total) default to strong scaling
  (--scaling strong: the fixed total split over the N GPUs).  Runs are sharded
  by hypercube range (the reference's partition rule, each split point
  snapped to the next cube start) and merged by one NCCL all-reduce per
  iteration.  Synthetic: the integrand is a closed-form function, nothing is
  loaded.
* a step = one full iteration (plan -> fused fill -> [all-reduce] ->
  results -> allocation -> refine) on device.  W warm-up iterations, then K
  timed iterations; L2 is flushed (256 MiB write) before every timed
  iteration, outside its CUDA-event window.
* value = sum over ranks of evaluations (plan.total) / max-over-ranks device
  time; e2e = the same metric through the public host-buffer call
  (vpb_iteration_host: H2D of the map, D2H of estimate/variance/evals/map).
* roofline: the fused fill kernel against the FP64 pipe (measured DFMA rate
  on this GPU); work per evaluation in FP64-pipe instruction equivalents by
  SURVEY.md §8(d)'s formula with the SASS-measured costs in COST below.
* cpu_baseline: the C oracle port (oracle/) on this host's cores, rank 0,
  N=1, bounded sample.  --impl reference: the same oracle as the reference
  arm (the reference is Python and cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# --------------------------------------------------------------- workloads --
# Roofline work per evaluation in FP64-pipe instruction equivalents, the
# formula of SURVEY.md §8(d): add/sub/mul count + c_div * divisions +
# c_exp * exps + c_cos * coss, with the costs read from the SASS of the
# device code (frozen here): an exactly rounded division is 3 FP64-pipe
# instructions (Markstein: DMUL + 2 DFMA, devmath.cuh div_exact), the device
# exp 18 (fast_exp_nonpos: 1 clamp + Cody-Waite 4 + degree-11 Horner 11 +
# 2 scaling), libdevice cos 16.  `flops` is SURVEY §8(d)'s FLOP count
# (add/sub/mul/div = 1) and `div` the divisions in it.  cfg3 counts the
# algorithm the device runs: the reference's windowed sum of ~632 centre
# terms (vp/integrands.py:154-182) by the blocked exact-factor recurrence of
# integrands.cuh ridge_window -- per 64-centre block one direct exp pair and
# 6 FLOP, per centre 3 FLOP (two products and the sum), the centres
# RN(i/999) staged once per CTA: sampling 44 + setup 23 + 10 blocks x 6 +
# 632 x 3 + accumulate 8 = 2031 FLOP, 9 divisions, 22 exps.
COST = {"div": 3, "exp": 18, "cos": 16}
CONFIGS = {
    "cfg1": dict(integrand="gaussian", dims=4, n_eval=10**6, ng=1000, flops=65, div=9, exp=1),
    # cfg2: the device's fma form (integrands.cuh VPB_MP_FMA) multiplies by
    # RN(1/(2 sigma^2)) and by norm/3 instead of SURVEY's 4 divisions and 3
    # norm products: integrand 75 FLOP (an fma = a mul + an add), 0 divisions
    "cfg2": dict(integrand="multipeak8", dims=8, n_eval=10**8, ng=1024, flops=175, div=16, exp=3,
                 survey=dict(flops=177, div=20, exp=3)),
    "cfg3": dict(integrand="ridge", dims=4, n_eval=10**8, ng=1024, flops=2031, div=9, exp=22,
                 survey=dict(flops=3227, div=9, exp=632)),
    "cfg4a": dict(integrand="genz_oscillatory6", dims=6, n_eval=10**9, ng=1024, flops=88, div=12,
                  cos=1),
    # cfg4b: the product of the 6 reciprocals is evaluated as one reciprocal
    # of the product (integrands.cuh): integrand 24 FLOP + 1 division
    "cfg4b": dict(integrand="genz_productpeak6", dims=6, n_eval=10**9, ng=1024, flops=101, div=13,
                  survey=dict(flops=105, div=18)),
    "cfg5": dict(integrand="gaussian20", dims=20, n_eval=4 * 10**9, ng=1024, flops=305, div=41,
                 exp=1),
    # the paper's own breakdown workload ("def": ng 1024,
    # 20 iterations; 1e10 evaluations = 5e8 per iteration): Roos & Arnold
    # 10-D, prod |4 x_j - 2| -- transform 110 (20 div) + integrand 30 +
    # accumulate 14
    "ra10": dict(integrand="roos_arnold", dims=10, n_eval=5 * 10**8, ng=1024, flops=154, div=20),
}
METRIC = "integrand evals/sec per iteration (1/2/4/8 B200) + % FP64 roofline vs host CPU ref"
UNIT = "evals/s"


def fp64_ops_per_eval(cfg) -> float:
    """add/sub/mul + c_div*div + c_exp*exp + c_cos*cos."""
    return (cfg["flops"] - cfg.get("div", 0) + COST["div"] * cfg.get("div", 0)
            + COST["exp"] * cfg.get("exp", 0) + COST["cos"] * cfg.get("cos", 0))


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled (every 50 ms) during the
    timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = ""

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)   # first sample lands before the timed region
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()

    def summary(self):
        rows = [[c.strip() for c in l.split(",")] for l in self.out.strip().splitlines()
                if l.strip()]
        rows = [r for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[5:9])
                          if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# -------------------------------------------------------------- CPU oracle --
def cpu_oracle_rate(cfg, n_eval_sample: int, iters: int = 2, workers: int | None = None):
    """Time the oracle's fill on host cores: evals/s of the last iteration."""
    import oracle as O
    workers = workers or os.cpu_count() or 1
    out = O.integrate(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], n_eval_sample,
                      max_it=iters, n_intervals=cfg["ng"], workers=workers)
    return out.evals[-1] / out.fill_seconds[-1], workers, out


def cpu_model() -> str:
    """The host CPU's model name (BASELINE.md §2 asks for it with the core count)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(cfg) -> dict:
    """The oracle on all host threads (the reported value) and on one thread
    (W = all cores and W = 1), same cube geometry at a bounded
    n_eval sample; fill time of iteration 2 only."""
    sample = int(os.environ.get("VPB_CPU_SAMPLE", cfg["n_eval"] // 10))
    # one thread gets a tenth of the sample (same geometry: the cube cap
    # binds), keeping the leg within seconds
    sample1 = max(10 ** 6, sample // 10)
    rate, cores, _ = cpu_oracle_rate(cfg, sample)
    rate1, _, _ = cpu_oracle_rate(cfg, sample1, workers=1)
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
            "sample": f"oracle (C port of vp/executor.parallel_fill, {cores} threads) "
                      f"iteration 2 of {cfg['integrand']} at n_eval={sample} (same cube "
                      f"geometry as n_eval={cfg['n_eval']}); fill time only",
            "single_thread": {"value": rate1, "unit": UNIT, "cores": 1,
                              "sample": f"iteration 2 at n_eval={sample1}, 1 thread"},
            "thread_speedup": rate / rate1 if rate1 > 0 else None}


# ------------------------------------------------------------------ arms --
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")   # rendezvous + host-side max; NCCL lives in the .so
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args, cfgname, cfg, world, rank):
    """--impl reference: the CPU oracle (port of the reference path) on all
    host threads, same metric/config; rank 0 only."""
    if rank != 0:
        return
    sample = int(os.environ.get("VPB_REF_SAMPLE", 10**7))
    import oracle as O
    workers = os.cpu_count() or 1
    # one oracle "step" = one iteration of the same geometry at n_eval = sample
    # (cube geometry identical: the 2^20 cube cap binds)
    out = O.integrate(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], sample,
                      max_it=args.warmup + args.steps, n_intervals=cfg["ng"], workers=workers)
    ev = out.evals[args.warmup:]
    secs = out.fill_seconds[args.warmup:]
    value = sum(ev) / sum(secs)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfgname}: {cfg['integrand']} d={cfg['dims']} "
                               f"ng={cfg['ng']}", "n_eval_per_iteration": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.warmup + args.steps} oracle iterations of "
                                   f"{cfg['integrand']} at n_eval={sample} (same cube geometry "
                                   f"as n_eval={cfg['n_eval']}); fill time only"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def per_function_loop(cfg, n_eval, warmup, steps):
    """vp/core.py:200-219 with every function replaced by its C entry point
    (ops.py: build_run_plan, parallel_fill -> vpb_fill_host, compute_results,
    update_evals_per_cube, smooth_and_damp, update_grid), host numpy arrays
    in and out; wall clock per iteration, host<->device bytes counted from
    the arrays each call moves."""
    import numpy as np

    from paper_2408_09229_b200 import ops
    from paper_2408_09229_b200.core import compute_n_strat
    dims, ng = cfg["dims"], cfg["ng"]
    ns = compute_n_strat(n_eval, dims)
    edges = np.tile(np.linspace(0.0, 1.0, ng + 1), (dims, 1))
    n_h = ops.update_evals_per_cube(np.zeros(ns ** dims), 0.0, n_eval)
    run_base, seed, batch = 0, 0, 1 << 20
    times, evals, h2d, d2h = [], 0, 0, 0
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        off = ops.build_run_plan(n_h)
        mw, mc, s1, s2, cnt = ops.parallel_fill(off, edges, ns, seed, batch, cfg["integrand"],
                                                run_base)
        i_it, v_it, d_h = ops.compute_results(s1, s2, cnt)
        n_h = ops.update_evals_per_cube(d_h, 0.75, n_eval)
        edges = ops.update_grid(edges, ops.smooth_and_damp(mw, mc, 0.5))
        t1 = time.perf_counter()
        total = int(off[-1])
        run_base += total
        if it >= warmup:
            times.append(t1 - t0)
            evals += total
            # fill: offsets + edges in; map (f64 + i64) and s1, s2 out;
            # results: s1, s2, counts in, d_h out; allocation: d_h in, n_h
            # out; plan: n_h in, offsets out; damp + grid: map in, damped
            # out, edges + damped in, edges out
            nc = ns ** dims
            h2d += 8 * (nc + 1) + 8 * edges.size + 24 * nc + 8 * nc + 8 * nc + 16 * mw.size \
                + 8 * edges.size + 8 * mw.size
            d2h += 16 * mw.size + 16 * nc + 8 * nc + 8 * nc + 8 * (nc + 1) + 8 * mw.size \
                + 8 * edges.size
    t = sum(times)
    return {"value": evals / t, "unit": UNIT, "ms_per_step": 1e3 * t / len(times),
            "steps": len(times), "h2d_bytes_per_step": h2d // len(times),
            "d2h_bytes_per_step": d2h // len(times),
            "path": "ops.build_run_plan -> ops.parallel_fill (vpb_fill_host, cached context) "
                    "-> ops.compute_results -> ops.update_evals_per_cube -> "
                    "ops.smooth_and_damp -> ops.update_grid, host numpy buffers, wall clock"}


def run_gpu(args, cfgname, cfg, world, rank, local):
    import numpy as np
    import torch

    import paper_2408_09229_b200 as P
    from paper_2408_09229_b200 import _native as N

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    # weak: fixed work per GPU (n_eval x N); strong: BASELINE's fixed total
    # (cfg4's 1e9 and cfg5's 4e9 per iteration split over the N GPUs)
    n_eval = cfg["n_eval"] * world if args.scaling == "weak" else cfg["n_eval"]
    steps, warmup = args.steps, args.warmup
    conf = P.IntegratorConfig(n_eval=n_eval, max_it=warmup + steps + 1,
                              n_intervals=cfg["ng"])
    integ = P.Integrator(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], conf, device=local,
                         distributed=(world > 1) or None, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # measured FP64 peak (the roofline denominator; MEASURED_PEAKS.json has none)
    peak = N.f64([0.0])
    import ctypes
    pk = ctypes.c_double()
    N.check(N.load().vpb_fp64_peak(local, ctypes.byref(pk)))
    peak_ops = pk.value

    # ---- device-resident loop
    integ.iterate(warmup)
    integ.sync()
    barrier(world)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(steps):
        flush.zero_()                         # L2 flush, outside the iteration's events
        integ.iterate(1)
    torch.cuda.synchronize(dev)
    clocks.stop()
    barrier(world)
    est, var, evals = integ.history()
    iter_ms, fill_ms = integ.timing_ms(warmup, steps)
    t_max = allreduce_max(iter_ms, world)
    evals_timed = int(np.sum(evals[warmup:warmup + steps]))   # plan.total is global
    value = evals_timed / (t_max * 1e-3)
    fill_ms_max = allreduce_max(fill_ms, world)

    # ---- e2e through the host-buffer C call (a fresh context, same workload)
    e_conf = P.IntegratorConfig(n_eval=n_eval, max_it=warmup + steps + 1,
                                n_intervals=cfg["ng"])
    e_integ = P.Integrator(cfg["integrand"], [(0.0, 1.0)] * cfg["dims"], e_conf, device=local,
                           distributed=(world > 1) or None)
    edges_host = N.f64(e_integ.edges())
    pinned_in = torch.from_numpy(edges_host).pin_memory().numpy()
    pinned_out = torch.empty(pinned_in.shape, dtype=torch.float64).pin_memory().numpy()
    for _ in range(warmup):
        e_integ.iteration_host(pinned_in, pinned_out)
        pinned_in[...] = pinned_out
    barrier(world)
    t0 = time.perf_counter()
    e_evals = 0
    for _ in range(steps):
        _, _, ev = e_integ.iteration_host(pinned_in, pinned_out)
        pinned_in[...] = pinned_out
        e_evals += ev
    t1 = time.perf_counter()
    e_time = allreduce_max(t1 - t0, world)
    e2e_value = e_evals / e_time
    h2d = pinned_in.nbytes
    d2h = pinned_out.nbytes + 8 + 8 + 8
    e_integ.close()

    # ---- the per-function binding: the reference's own
    # iteration loop kept in the host language, each function on the path a
    # stateless C call with host buffers (ops.py = the ctypes stub), so the
    # plan offsets, the map and the accumulators cross PCIe every iteration
    per_function = None
    if world == 1 and not args.no_per_function:
        per_function = per_function_loop(cfg, n_eval, warmup, min(steps, 5))

    layout = integ.fill_layout()
    fx = integ.fx_stats()
    fx["mode"] = "fixed point (per-interval predicted scale)" if fx["enabled"] else "f64 CAS"
    if rank == 0:
        ops = fp64_ops_per_eval(cfg)
        # fill kernel: per-rank evaluations = its shard of each plan
        evals_per_rank = evals_timed / world
        achieved = ops * evals_per_rank / (fill_ms_max * 1e-3)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "fill_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(cfgname)
            except Exception:
                traffic = None
        # SURVEY 8(d)'s issue-bound variant: the fill's executed instructions
        # per evaluation (ncu smsp__inst_executed.sum of one fill launch,
        # profiles/fill_traffic.json "inst_per_eval") at the measured rate,
        # against 4 warp-instructions per clock per SM at the sampled clock
        issue = None
        try:
            ipe = json.load(open(tp)).get("inst_per_eval", {}).get(cfgname)
        except Exception:
            ipe = None
        clk = clocks.summary()
        mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz")
        if ipe and mhz:
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            warp_ips = evals_per_rank / (fill_ms_max * 1e-3) * ipe / 32.0
            ipeak = sms * 4 * mhz * 1e6
            issue = {"inst_per_eval": ipe, "achieved": warp_ips / 1e12, "peak": ipeak / 1e12,
                     "unit": "T warp-instr/s", "frac": warp_ips / ipeak,
                     "source": "lane instructions per evaluation from ncu (profiles/"
                               "fill_traffic.json); peak = 4 issue slots/clk/SM x SMs x "
                               "sampled SM clock"}
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline(cfg)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": t_max / steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (closed-form integrand, nothing loaded)",
            "config": {"workload": f"{cfgname}: {cfg['integrand']} d={cfg['dims']}, "
                                   f"n_eval={cfg['n_eval']:.0e}/iter"
                                   f"{'/GPU' if args.scaling == 'weak' else ' in total'}, "
                                   f"ng={cfg['ng']}",
                       "n_eval_per_iteration": n_eval, "n_strat": integ.n_strat,
                       "n_cubes": integ.n_cubes, "evals_per_step": evals_timed / steps,
                       "parallelism": f"hypercube-aligned run shards over {world} GPU(s), "
                                      f"one NCCL all-reduce per iteration",
                       "l2": "flushed (256 MiB write) before every timed iteration",
                       "fill_layout": layout["layout"], "record_chunks": layout["chunks"]},
            "roofline": {"bound": "fp64", "achieved": achieved / 1e12,
                         "peak": peak_ops / 1e12, "unit": "TFLOP/s",
                         "frac": achieved / peak_ops, "traffic": traffic,
                         "kernel": "vpb::fill_kernel (fused Philox->map->integrand->histograms)",
                         "convention": "FP64-pipe instruction equivalents per SURVEY 8(d): "
                                       "add/sub/mul=1, exact div=3, exp=18, cos=16 (SASS "
                                       "counts), of the operations the device algorithm "
                                       "performs (fma = mul + add); peak = measured DFMA "
                                       "rate on this GPU (vpb_fp64_peak)",
                         "ops_per_eval": ops,
                         # the same rate with SURVEY 8(d)'s per-evaluation
                         # figure (the reference's operation count) where the
                         # device runs fewer operations (cfg2, cfg3, cfg4b);
                         # `frac` above never credits work the device skips
                         "frac_survey_figure": achieved / peak_ops
                         * fp64_ops_per_eval(cfg.get("survey", cfg)) / ops,
                         "fill_kernel_ms_per_step": fill_ms_max / steps,
                         "fill_share_of_step": fill_ms_max / t_max, "issue": issue},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "per_function_binding": per_function,
            "gpu_launches": layout["launches_per_iteration"] * steps,
            "clocks": clk,
            "estimates": {"last": float(est[-1]), "sigma_last": float(np.sqrt(var[-1]))},
            # fixed-point interval histograms (fill.cuh LAYOUT_FX): iterations
            # filled in fixed point, redone in f64, values spilled to f64
            "histograms": fx,
        }
        print(json.dumps(line), flush=True)
    integ.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-per-function", action="store_true",
                    help="skip the per-function-binding measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: n_eval per GPU; strong: n_eval in total (default: strong for "
                         "BASELINE's multi-GPU configs cfg4a/cfg4b/cfg5, weak otherwise)")
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = "strong" if args.config in ("cfg4a", "cfg4b", "cfg5") else "weak"
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, args.config, cfg, world, rank)
    else:
        run_gpu(args, args.config, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
