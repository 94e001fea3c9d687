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
