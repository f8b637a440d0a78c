"""Multi-GPU plumbing for the sharded points solve.

One process per GPU; ``torch.distributed`` is only the bootstrap channel: rank
0 asks the library for an NCCL unique id, broadcasts its 128 bytes over the
existing process group (gloo or nccl), and every rank builds the library's own
communicator (``lsk_comm_create``) that the solver uses on its CUDA stream.

Sharding designs (``lsk_solve_points_f32``, include/lsk.h): column partials
(default; rank r owns a slab of whole 2048-point chunks of the source cloud,
the per-column partials of its rows are allgathered and merged by the top of a
fixed tree), allreduce (the stale sums by ncclAllReduce) and owner computes
(rank r owns rows ``[r ceil(n/P), ...)`` for f and columns ``[r ceil(m/P), ...)``
for g, potential slabs allgathered). Batched independent problems are split
across ranks instead (``split_batch``), with no communication at all.
"""

import ctypes

from . import _lib

__all__ = ["Communicator", "shard_bounds", "split_batch"]


def shard_bounds(n, world, rank):
    """[lo, hi) of the rows rank ``rank`` of ``world`` owns (the library's rule)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * n // world, (rank + 1) * n // world


def split_batch(B, world, rank):
    """Contiguous share of B independent problems for one rank (config C5:
    256 problems over 8 GPUs = 32 each); sizes differ by at most one."""
    return shard_bounds(B, world, rank)


def broadcast_unique_id(group=None):
    """NCCL unique id from rank 0 to every rank over torch.distributed."""
    import torch
    import torch.distributed as dist

    nbytes = _lib.load().lsk_nccl_unique_id_bytes()
    buf = ctypes.create_string_buffer(nbytes)
    if dist.get_rank(group) == 0:
        _lib.call("lsk_nccl_unique_id", buf)
    t = torch.tensor(list(buf.raw), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


class Communicator:
    """The library's NCCL communicator for this rank (one GPU per rank)."""

    def __init__(self, uid, world, rank):
        self.world, self.rank = int(world), int(rank)
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(uid), len(uid))
        _lib.call("lsk_comm_create", buf, self.world, self.rank, ctypes.byref(h))
        self.handle = h.value

    @classmethod
    def from_torch_distributed(cls, group=None):
        import torch.distributed as dist

        uid = broadcast_unique_id(group)
        return cls(uid, dist.get_world_size(group), dist.get_rank(group))

    def close(self):
        if self.handle:
            _lib.call("lsk_comm_destroy", ctypes.c_void_p(self.handle))
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
