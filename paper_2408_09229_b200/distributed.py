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
