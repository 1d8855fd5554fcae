"""Multi-process (gloo, world size 2) checks of the sharding logic on CPU: angle-row shards of
W whose partial adjoints, summed by an all-reduce, equal the full adjoint; slice shards that
cover every slice exactly once. The per-rank compute is the fp64 oracle (CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_07497_b200.distributed import angle_blocks, slice_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    n, A, nb = 32, 13, 33
    a0, a1 = angle_blocks(A, world)[rank]
    angles = np.arange(A) * np.pi / A
    g_loc = O.Geometry(n=n, n_angles=a1 - a0, n_b=nb, win_lo=-2, win_hi=3, tau=3 / n ** 2, angles=angles[a0:a1])
    rng = np.random.default_rng(5)
    s_full = rng.standard_normal(A * nb) + 1j * rng.standard_normal(A * nb)
    part = O.type1(g_loc, s_full[a0 * nb:a1 * nb])
    t = torch.from_numpy(np.stack([part.real, part.imag]).copy())
    dist.all_reduce(t)
    # the normal operator of a real image: forward on the local block, adjoint, all-reduce
    u = rng.standard_normal((n, n))
    nu = O.type1(g_loc, O.type2(g_loc, u)).real
    tn = torch.from_numpy(nu.copy())
    dist.all_reduce(tn)
    if rank == 0:
        out.put((t.numpy(), tn.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_angle_blocks_partition():
    for A in (13, 90, 360):
        for w in (1, 2, 3, 8):
            if A < w:
                continue
            b = angle_blocks(A, w)
            assert b[0][0] == 0 and b[-1][1] == A
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1


def test_slice_shards_cover_once():
    for S in (1, 7, 256):
        for w in (1, 2, 4, 8):
            seen = [i for r in range(w) for i in slice_shard(S, w, r)]
            assert seen == list(range(S))


def test_gloo_world2_angle_shards_sum_to_full_adjoint():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    adj, nu = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, A, nb = 32, 13, 33
    g = O.Geometry(n=n, n_angles=A, n_b=nb, win_lo=-2, win_hi=3, tau=3 / n ** 2)
    rng = np.random.default_rng(5)
    s_full = rng.standard_normal(A * nb) + 1j * rng.standard_normal(A * nb)
    full = O.type1(g, s_full)
    assert np.allclose(adj[0] + 1j * adj[1], full, rtol=1e-12, atol=1e-9)
    u = rng.standard_normal((n, n))
    assert np.allclose(nu, O.apply_normal_real(g, u), rtol=1e-10, atol=1e-8)
