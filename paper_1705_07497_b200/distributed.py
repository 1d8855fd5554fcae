"""Multi-GPU partitioning of the hot path, one process per GPU.

* Independent slices (config 4): `slice_shard` — contiguous slice ranges per rank, no collective.
* One large slice (config 5): `angle_blocks` — W is row-sharded by contiguous angle blocks; each
  rank owns the samples of its block, and the partial type-1 images are summed across ranks by
  an all-reduce inside the library after every adjoint (`make_sharded_backend` wires an NCCL
  communicator, bootstrapped through torch.distributed).
"""
from __future__ import annotations


def angle_blocks(n_angles: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [begin, end) angle ranges, one per rank (every rank non-empty)."""
    if world < 1 or n_angles < world:
        raise ValueError("need at least one angle per rank")
    base, extra = divmod(n_angles, world)
    out, a = [], 0
    for r in range(world):
        k = base + (1 if r < extra else 0)
        out.append((a, a + k))
        a += k
    return out


def slice_shard(n_slices: int, world: int, rank: int) -> range:
    """Contiguous slice range of `rank` (ceil split; trailing ranks may be shorter or empty)."""
    per = (n_slices + world - 1) // world
    lo = min(n_slices, rank * per)
    return range(lo, min(n_slices, lo + per))


def make_sharded_backend(geom, rank: int, world: int, device: int, group=None, **kw):
    """Direct backend owning this rank's angle block, with an NCCL all-reduce of the partial
    adjoint images across `world` ranks (communicator id broadcast via torch.distributed)."""
    import torch.distributed as dist

    from .tomo import NormalBackend, nccl_unique_id
    a0, a1 = angle_blocks(geom.n_angles, world)[rank]
    op = NormalBackend(geom, "direct", device=device, angle_block=(a0, a1), **kw)
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        op.attach_nccl(obj[0], world, rank)
    return op
