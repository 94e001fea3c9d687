"""Multi-GPU plumbing: one process per GPU, torch.distributed for rendezvous.

The NCCL communicator used by the hot path lives inside libvegas_b200.so
(the per-iteration all-reduce is enqueued on the context's stream between
the fill and the replicated update).  torch.distributed only carries the
128-byte NCCL unique id from rank 0 to the other ranks.
"""

from __future__ import annotations

import ctypes


def nccl_unique_id_broadcast(lib) -> bytes:
    import torch.distributed as dist

    from . import _native as N

    buf = ctypes.create_string_buffer(128)
    if dist.get_rank() == 0:
        N.check(lib.vpb_nccl_unique_id(buf), "vpb_nccl_unique_id")
    obj = [bytes(buf.raw) if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def host_allreduce_callback():
    """A vpb_allreduce_fn that all-reduces the library's pinned host staging
    buffers in place with torch.distributed (the process group's backend,
    e.g. gloo): the exchange path for ranks without NCCL (tests: several
    ranks on one GPU).  Keep the returned object alive with the context."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import _native as N

    ops = {N.VPB_OP_SUM: dist.ReduceOp.SUM, N.VPB_OP_MAX: dist.ReduceOp.MAX}
    types = {N.VPB_DT_F64: ctypes.c_double, N.VPB_DT_I64: ctypes.c_int64}

    def fn(_user, buf, count, dtype, op):
        try:
            arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(types[dtype])),
                                        shape=(int(count),))
            dist.all_reduce(torch.from_numpy(arr), op=ops[op])   # in place, shares memory
            return 0
        except Exception:   # reported by the library as an exchange failure
            return 1

    return N.ALLREDUCE_FN(fn)


def partition_runs(total: int, k: int):
    """vp/executor.py:41-57: k contiguous ranges, the first total % k get +1.
    (The device plan kernel applies the same rule per rank.)"""
    if total < 0 or k < 1:
        raise ValueError("need total >= 0 and k >= 1")
    q, rem = divmod(total, k)
    out, start = [], 0
    for i in range(k):
        size = q + (1 if i < rem else 0)
        out.append((start, start + size))
        start += size
    return out
