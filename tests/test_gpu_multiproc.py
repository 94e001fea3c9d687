"""Multi-process runs of the sharded data path on the GPU: one process per
rank (torch.distributed, gloo), every rank's context on cuda:0 (this build
has one GPU; NCCL refuses two ranks on one device, so the merge here is the
host all-reduce that stands in for the device one).  Each rank fills its
shard of the run range, split by the reference's partition rule
(vp/executor.py:41-57) on the device, and the summed accumulators must equal
the whole single-process fill -- exactly for the counts, to the cube-sum
tolerance for the weights.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = dict(n_eval=300_000, max_it=3, n_intervals=64, seed=21, batch_size=4096)
RUN_BASE = 123_457


def _accumulate(world, rank):
    import paper_2408_09229_b200 as P
    with P.Integrator("multipeak8", [(0.0, 1.0)] * 8, P.IntegratorConfig(**CFG),
                      distributed=False) as it:
        if world > 1:
            it.set_shard(world, rank)
        it.fill(RUN_BASE)
        return it.accumulators()


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        parts = _accumulate(world, rank)
        bufs = [torch.from_numpy(np.ascontiguousarray(a)) for a in parts]
        for b in bufs:
            dist.all_reduce(b)
        if rank == 0:
            whole = _accumulate(1, 0)
            m = [b.numpy() for b in bufs]
            ok = (np.array_equal(m[1], whole[1]) and np.array_equal(m[4], whole[4])
                  and np.allclose(m[0], whole[0], rtol=1e-12, atol=0)
                  and np.allclose(m[2], whole[2], rtol=1e-12, atol=1e-290)
                  and np.allclose(m[3], whole[3], rtol=1e-12, atol=1e-290)
                  and int(m[4].sum()) == int(whole[4].sum()) > 0)
            q.put(("ok", bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # surfaced to the parent
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}"))


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_shards_merge_to_whole(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 17 + (os.getpid() % 400)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    for p in procs:
        if p.is_alive():   # a rank died and left its peer waiting in the all-reduce
            p.kill()
    kind, val = q.get(timeout=30)
    assert kind == "ok", val
    assert val is True
    assert all(p.exitcode == 0 for p in procs)


# ----------------------------------------------- the whole iteration, world > 1
# Every rank runs full iterations (plan -> its hypercube-aligned shard of the
# fill -> exchange -> replicated update) with the exchange through the host
# all-reduce callback over gloo (vpb_attach_exchange; the same three
# reductions as the NCCL group, incl. the control word).

IT_CFG = dict(n_eval=200_000, max_it=4, n_intervals=128, seed=9, batch_size=4096)
# exponential exp(sum x^2) with the last axis on (0, 30): the top stratum of that
# axis (x > 26.5) overflows to inf -- its cubes are the last third of the plan, i.e. only the
# last rank's shard fails (vp/executor.py:119-127)
NF_BOUNDS = [(0.0, 1.0)] * 9 + [(0.0, 30.0)]


FX_CFG = dict(n_eval=2_000_000, max_it=5, n_intervals=1024, seed=9)


def _iterate(bounds, name, distributed, cfg=None):
    import paper_2408_09229_b200 as P
    cfg = cfg or IT_CFG
    with P.Integrator(name, bounds, P.IntegratorConfig(**cfg), device=0,
                      distributed=distributed, exchange="host") as it:
        it.iterate(cfg["max_it"])
        try:
            est, var, ev = it.history()
        except P.NonFiniteIntegrandError as e:
            return ("nonfinite", [float(v) for v in e.point], float(e.value), int(e.run_index),
                    it.world, it.rank)
        return ("ok", est.tolist(), var.tolist(), ev.tolist(), it.edges().tolist(), it.world)


def _iter_worker(rank, world, port, case, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        if case == "nonfinite":
            q.put((rank, _iterate(NF_BOUNDS, "exponential", True)))
        elif case == "fx":
            os.environ["VPB_HIST_FIXED"] = "1"
            q.put((rank, _iterate([(0.0, 1.0)] * 6, "genz_productpeak6", True, FX_CFG)))
        else:
            q.put((rank, _iterate([(0.0, 1.0)] * 8, "multipeak8", True)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced to the parent
        q.put((rank, ("error", f"{type(e).__name__}: {e}")))


def _run_ranks(world, case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + world * 31 + (os.getpid() % 300) + {"nonfinite": 7, "fx": 13}.get(case, 0)
    procs = [ctx.Process(target=_iter_worker, args=(r, world, port, case, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=300)
        out[r] = res
    for p in procs:
        p.join(60)
        if p.is_alive():
            p.kill()
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_iterations_match_single(world):
    out = _run_ranks(world, "ok")
    single = _iterate([(0.0, 1.0)] * 8, "multipeak8", False)
    assert single[0] == "ok"
    for r in range(world):
        kind, est, var, ev, edges, w = out[r]
        assert kind == "ok" and w == world, out[r]
        assert ev == single[3]                              # plan.total per iteration, exact
        np.testing.assert_allclose(est, single[1], rtol=1e-10)
        np.testing.assert_allclose(var, single[2], rtol=1e-8)
        np.testing.assert_allclose(edges, single[4], rtol=1e-12, atol=0)
        # the replicated update leaves every rank with the same map, bitwise
        assert edges == out[0][4]


def test_multiprocess_iterations_with_fixed_point_histograms(monkeypatch):
    """Each rank fills its shard with the fixed-point histograms (its own
    proof-or-redo), the host exchange merges the per-rank sums, and the
    replicated update (and its scale predictions) stays bitwise equal across
    ranks."""
    out = _run_ranks(2, "fx")
    monkeypatch.setenv("VPB_HIST_FIXED", "1")
    single = _iterate([(0.0, 1.0)] * 6, "genz_productpeak6", False, FX_CFG)
    assert single[0] == "ok"
    for r in range(2):
        kind, est, var, ev, edges, w = out[r]
        assert kind == "ok" and w == 2, out[r]
        assert ev == single[3]
        np.testing.assert_allclose(est, single[1], rtol=1e-10)
        np.testing.assert_allclose(var, single[2], rtol=1e-8)
        np.testing.assert_allclose(edges, single[4], rtol=1e-12, atol=0)
        assert edges == out[0][4]


def test_multiprocess_nonfinite_raises_on_every_rank():
    # only the last rank's shard evaluates to inf; every rank must raise the
    # same NonFiniteIntegrandError (the lowest failing run of the iteration,
    # its point and value) as the single-process run
    out = _run_ranks(2, "nonfinite")
    single = _iterate(NF_BOUNDS, "exponential", False)
    assert single[0] == "nonfinite"
    for r in range(2):
        assert out[r][0] == "nonfinite", out[r]
        assert out[r][1:4] == single[1:4], (out[r], single)
        assert out[r][4:] == (2, r)
