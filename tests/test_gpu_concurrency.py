"""One op serving two host threads on two CUDA streams at once (built
operators are immutable and shareable; concurrent solves on separate state are safe). Each call
leases its own workspace, so the concurrent results must equal the serial ones bit for bit."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def _geom(T):
    return T.Geometry(n=256, n_angles=60, n_b=257, win_lo=-2, win_hi=3, tau=3 / 256 ** 2)


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_concurrent_applies_on_one_op_bit_identical(T, prec):
    op = T.make_direct_backend(_geom(T), precision=prec, max_batch=3)
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    gen = torch.Generator(device="cuda").manual_seed(5)
    us = [torch.randn(3, 256, 256, dtype=cdt, device="cuda", generator=gen) for _ in range(2)]
    serial = [op.apply_normal(u).clone() for u in us]
    torch.cuda.synchronize()
    outs = [[None] * 25 for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]

    def worker(k):
        def f():
            with torch.cuda.stream(streams[k]):
                for i in range(25):
                    outs[k][i] = op.apply_normal(us[k])
                streams[k].synchronize()
        return f

    _run_threads([worker(0), worker(1)])
    for k in range(2):
        for o in outs[k]:
            assert torch.equal(o, serial[k])


def test_concurrent_split_bregman_on_one_op_bit_identical(T):
    from oracle import oracle as O
    g = _geom(T)
    og = O.Geometry(n=g.n, n_angles=g.n_angles, n_b=g.n_b, win_lo=g.win_lo, win_hi=g.win_hi, tau=g.tau)
    fs = [O.synthesize(og, O.random_ellipses(g.n, 10, s), 0.01, s)[0] for s in (1, 2)]
    op = T.make_direct_backend(g, precision="f64")
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=6, cg_steps_per_update=5, update_tol_rel=0.0)
    fd = [torch.from_numpy(f).cuda() for f in fs]
    serial = [op.split_bregman(f, cfg)[0].clone() for f in fd]
    res = [[None] * 3 for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]

    def worker(k):
        def f():
            with torch.cuda.stream(streams[k]):
                for i in range(3):
                    res[k][i] = op.split_bregman(fd[k], cfg)[0]
                streams[k].synchronize()
        return f

    _run_threads([worker(0), worker(1)])
    for k in range(2):
        for r in res[k]:
            assert torch.equal(r, serial[k])


def test_concurrent_cg_and_apply_mixed(T):
    """A CG solve and applies interleaved on one op from two threads (different entry points,
    different batch sizes, so the two workspaces are sized and captured differently)."""
    g = _geom(T)
    op = T.make_direct_backend(g, precision="f64", max_batch=2)
    gen = torch.Generator(device="cuda").manual_seed(9)
    rhs = torch.randn(256, 256, dtype=torch.float64, device="cuda", generator=gen)
    u = torch.randn(2, 256, 256, dtype=torch.float64, device="cuda", generator=gen)
    x_ser, _ = op.cg(rhs, alpha=1.0, lambda_=0.5, steps=12)
    a_ser = op.apply_normal_real(u)
    torch.cuda.synchronize()
    xs, As = [], []
    streams = [torch.cuda.Stream() for _ in range(2)]

    def solve():
        with torch.cuda.stream(streams[0]):
            for _ in range(4):
                xs.append(op.cg(rhs, alpha=1.0, lambda_=0.5, steps=12)[0])
            streams[0].synchronize()

    def apply():
        with torch.cuda.stream(streams[1]):
            for _ in range(10):
                As.append(op.apply_normal_real(u))
            streams[1].synchronize()

    _run_threads([solve, apply])
    assert all(torch.equal(x, x_ser) for x in xs)
    assert all(torch.equal(a, a_ser) for a in As)
