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


_CUDART = None


def _cudart():
    """The CUDA runtime torch loaded (host-exchange hook: stream sync + plain copies)."""
    global _CUDART
    if _CUDART is None:
        import ctypes

        import torch
        torch.cuda.init()
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _CUDART = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _CUDART is None:
            raise RuntimeError("libcudart not found")
        _CUDART.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]
        _CUDART.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    return _CUDART


def host_allreduce_hook(f64: bool, group=None):
    """An all-reduce for `NormalBackend.set_allreduce` (tomo_op_set_allreduce) that sums the
    partial adjoint images through the host with torch.distributed on `group` (e.g. gloo):
    synchronise the op's stream, copy device -> host, all-reduce, copy back. For ranks without an
    NCCL path between their devices; an op with a host hook runs its solver loops without CUDA
    graphs (the hook cannot be captured)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    rt = _cudart()
    dtype = np.float64 if f64 else np.float32
    esz = 8 if f64 else 4
    H2D, D2H = 1, 2

    def fn(buf, count, stream):
        if rt.cudaStreamSynchronize(stream) != 0:
            raise RuntimeError("cudaStreamSynchronize failed")
        host = np.empty(count, dtype)
        if rt.cudaMemcpy(host.ctypes.data, buf, count * esz, D2H) != 0:
            raise RuntimeError("cudaMemcpy D2H failed")
        t = torch.from_numpy(host)
        dist.all_reduce(t, group=group)
        if rt.cudaMemcpy(buf, host.ctypes.data, count * esz, H2D) != 0:
            raise RuntimeError("cudaMemcpy H2D failed")

    return fn


def make_sharded_backend(geom, rank: int, world: int, device: int, group=None, exchange: str = "nccl", **kw):
    """Direct backend owning this rank's angle block whose partial adjoint images are summed
    across `world` ranks after every type-1 transform: exchange="nccl" builds an NCCL
    communicator inside the library (id broadcast via torch.distributed) and keeps the solver
    loops in CUDA graphs; exchange="host" sums through torch.distributed on `group` (gloo)."""
    import torch.distributed as dist

    from .tomo import NormalBackend, nccl_unique_id
    a0, a1 = angle_blocks(geom.n_angles, world)[rank]
    op = NormalBackend(geom, "direct", device=device, angle_block=(a0, a1), **kw)
    if world > 1 or exchange == "host":
        if exchange == "nccl":
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            op.attach_nccl(obj[0], world, rank)
        elif exchange == "host":
            op.set_allreduce(host_allreduce_hook(op.f64, group))
        else:
            raise ValueError(f"unknown exchange {exchange!r}")
    return op
