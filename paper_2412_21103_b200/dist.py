"""Multi-process plumbing around the C ABI's dist context.

The library does the distributed work itself (include/nw.h "distributed context"):
nw_ctx_set_dist joins an NCCL communicator, and nw_align_batch(_dev) on such a
context aligns this rank's cost-balanced range (nw_batch_partition) and gathers
every range with one group of in-place NCCL broadcasts. This module only:
  - shares the 128-byte NCCL id from rank 0 over an existing torch.distributed
    group (share_unique_id / init_dist_context),
  - launches one process per GPU when the caller did not (launch), and
  - exposes the partition for tests (partition = nw_batch_partition).
Host logic only: no scores are computed here.
"""
from __future__ import annotations

import os
import socket

from . import nw as _nw


def share_unique_id(group=None) -> bytes:
    """Rank 0's nw_dist_unique_id, broadcast to every rank of `group` (any backend)."""
    import torch.distributed as dist
    obj = [_nw.nw_dist_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_dist_context(ctx, group=None) -> None:
    """Attach ctx (one per process, on this rank's GPU) to a communicator spanning
    `group` (collective)."""
    import torch.distributed as dist
    uid = share_unique_id(group)
    ctx.set_dist(dist.get_rank(group), dist.get_world_size(group), uid)


def partition(offs, pairs, world: int):
    """bounds[0..world]: rank r aligns tasks [bounds[r], bounds[r+1]) (include/nw.h)."""
    return _nw.nw_batch_partition(offs, pairs, world)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _child(local_rank, world, port, fn, args):
    os.environ.update(RANK=str(local_rank), LOCAL_RANK=str(local_rank), WORLD_SIZE=str(world),
                      LOCAL_WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    fn(*args)


def launch(nprocs: int, fn, args=()) -> None:
    """Run fn(*args) in nprocs fresh processes, one per rank, with the torchrun
    environment (RANK, LOCAL_RANK, WORLD_SIZE, MASTER_ADDR=127.0.0.1, MASTER_PORT)
    set; raises if any rank fails."""
    import torch.multiprocessing as mp
    mp.spawn(_child, args=(nprocs, free_port(), fn, args), nprocs=nprocs, join=True)
