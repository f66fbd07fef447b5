"""Multi-GPU partitioning (one process per GPU).  The partition rule is the
C-ABI's own (qf_shard_range, the function csrc/capi.cpp's sharded
qf_energy_grad_batch uses), so host code and tests share one implementation.

Batch sharding: rank r owns parameter-set rows [B r / p, B (r+1) / p); every
other row of the [B x (1+P)] result buffer stays zero, so one all-reduce(sum)
reconstructs the full result bitwise (x + 0 = x): results never depend on the
GPU count (reference include/qforge/parallel.hpp:9-10).
Term sharding (single large state): rank r owns Hamiltonian terms
[T r / p, T (r+1) / p); energy and gradient are linear in H, so the all-reduce
sums the partial results (equal to the 1-GPU result up to rounding).
"""
from __future__ import annotations


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) owned by `rank` of `world` (qf_shard_range; host-only call)."""
    import ctypes

    from . import _lib

    b, e = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().qf_shard_range(int(count), int(rank), int(world), ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def init_engine_comm(ctx, group=None) -> None:
    """Create the engine's NCCL communicator from an initialised torch.distributed
    process group (rank 0 makes the id, broadcast_object_list ships it)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        ctx.set_comm(0, 1, None)
        return
    obj = [ctx.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.set_comm(rank, world, obj[0])
