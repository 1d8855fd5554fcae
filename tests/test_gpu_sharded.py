"""Angle-block sharding of one slice (config c5's multi-GPU path) run by two real
processes: each rank builds the product's op over its angle block of W (tomo_op_create with
angle_begin/end), and the partial adjoint images are summed after every type-1 transform through
tomo_op_set_allreduce with a gloo-backed host hook (distributed.host_allreduce_hook). Both ranks
share the one GPU of the box; their kernels never wait on each other (the exchange is on the
host), so this is a faithful 2-rank run of the sharded apply / CG / Chambolle-Pock, compared
with the unsharded op at 1e-10 (fp64). Reference: SPEC.md:296 (per-angle blocks, then a
reduction for the adjoint)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10
GEOM = dict(n=128, n_angles=31, n_b=129, oversample=4, win_lo=-2, win_hi=3)
CP = dict(alpha=1e-2, lambda_=1e-2, tau_cp=0.35, sigma_cp=0.35, theta=1.0, iters=2, cg_steps=6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(T):
    from oracle import oracle as O
    g = T.Geometry(**GEOM)
    og = O.Geometry(**GEOM, tau=g.tau)
    ph = O.random_ellipses(g.n, 10, 77)
    f, _ = O.synthesize(og, ph, 0.01, 77)
    rng = np.random.default_rng(3)
    u = rng.standard_normal((g.n, g.n))
    return g, f, u


def _run(op, T, f, u):
    dev = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dt)).cuda()  # noqa: E731
    out = {}
    out["apply"] = op.apply_normal_real(dev(u, np.float64)).cpu().numpy()
    out["backproject"] = op.backproject(dev(f, np.complex128), alpha=2.0).cpu().numpy()
    x, _ = op.cg(dev(u, np.float64), alpha=1.0, lambda_=0.5, shift=0.0, steps=8)
    out["cg"] = x.cpu().numpy()
    out["cp"] = op.chambolle_pock(dev(f, np.complex128), **CP).cpu().numpy()
    out["tikhonov"] = op.tikhonov(dev(f, np.complex128), alpha=1.0, steps=6).cpu().numpy()
    return out


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1705_07497_b200 as T
        from paper_1705_07497_b200.distributed import angle_blocks, make_sharded_backend
        g, f, u = _inputs(T)
        a0, a1 = angle_blocks(g.n_angles, world)[rank]
        op = make_sharded_backend(g, rank, world, device=0, exchange="host", precision="f64")
        assert op.info.n_angles_local == a1 - a0
        res = _run(op, T, f[a0 * g.n_b:a1 * g.n_b], u)
        if rank == 0:
            q.put(res)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put(repr(e))
        raise


def test_two_rank_angle_sharded_matches_unsharded():
    import torch.multiprocessing as mp

    import paper_1705_07497_b200 as T
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    assert all(p.exitcode == 0 for p in procs)
    g, f, u = _inputs(T)
    full = _run(T.make_direct_backend(g, precision="f64"), T, f, u)
    for k, v in full.items():
        err = float(np.linalg.norm(res[k] - v) / np.linalg.norm(v))
        print(f"sharded x2 vs unsharded {k}: rel-L2 {err:.3e}")
        assert err <= TOL, (k, err)
