"""Edge cases of the device path the reference also defines: zero and non-finite inputs, even
n_b (broken conjugation symmetry -> split_bregman_tv's leak check, solver.cpp:236-247),
batches beyond max_batch, empty batches through the C ABI."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import rel
from tests.test_gpu_parity import GEOMS, cuda, pgeom

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def test_zero_input_gives_exact_zero(T):
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    for prec in ("f32", "f64"):
        op = T.make_direct_backend(pgeom(T, og), precision=prec)
        z = cuda(np.zeros((og.n, og.n)), True, prec == "f64")
        assert not op.apply_normal(z).abs().max().item()
        assert not op.forward(z).abs().max().item()


def test_nonfinite_iterate_raises_numerical_error(T):
    og = O.Geometry(**GEOMS["ref_msp3"])
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    rhs = np.ones((og.n, og.n))
    rhs[3, 4] = np.nan
    with pytest.raises(T.NumericalError):
        op.cg(cuda(rhs, False, True), alpha=1.0, lambda_=1.0, steps=3)
    f = np.zeros(og.P, np.complex128)
    f[5] = np.inf
    cfg = T.SolverConfig(alpha=1.0, lambda_=1.0, max_bregman_iters=2, cg_steps_per_update=2, update_tol_rel=0.0)
    with pytest.raises(T.NumericalError):
        op.split_bregman(cuda(f, True, True), cfg)


def test_even_nb_breaks_conjugation_symmetry(T):
    """n_b even: the point set is not symmetric under k -> -k, so Im(N u) leaks for real u
    (4.8e-2 at n = 64) while odd n_b keeps it at the window's accuracy; the
    split-Bregman leak diagnostic (probe = ones, solver.cpp:236-247) matches the oracle."""
    rng = np.random.default_rng(9)
    u = rng.standard_normal((64, 64))
    leak = {}
    for nb in (64, 65):
        og = O.Geometry(n=64, n_angles=50, n_b=nb, win_lo=-3, win_hi=3)
        op = T.make_direct_backend(pgeom(T, og), precision="f64")
        out = op.apply_normal(cuda(u, True, True)).cpu().numpy()
        leak[nb] = np.linalg.norm(out.imag) / np.linalg.norm(out)
        ref = O.apply_normal(og, u.astype(np.complex128))
        assert abs(leak[nb] - np.linalg.norm(ref.imag) / np.linalg.norm(ref)) < 1e-9
        cfg = T.SolverConfig(alpha=1.0, lambda_=1.0, max_bregman_iters=1, cg_steps_per_update=1, update_tol_rel=0.0)
        f = np.zeros(og.P, np.complex128)
        _, tr = op.split_bregman(cuda(f, True, True), cfg)
        _, _, rtr = O.split_bregman(og, f, backend=0, alpha=1.0, lam=1.0, max_iters=1, cg_steps=1)
        ref_leak = rtr.imag_leakage
        assert abs(tr[0].imag_leakage - ref_leak) <= 1e-9 + 1e-6 * ref_leak
    assert leak[64] > 1e-2 > 1e-3 > leak[65]


def test_batch_beyond_max_batch_grows(T):
    og = O.Geometry(**GEOMS["ref_msp3"])
    op = T.make_direct_backend(pgeom(T, og), precision="f64", max_batch=1)
    rng = np.random.default_rng(3)
    u = rng.standard_normal((5, og.n, og.n)) + 1j * rng.standard_normal((5, og.n, og.n))
    out = op.apply_normal(cuda(u, True, True)).cpu().numpy()
    for b in (0, 4):
        assert rel(out[b].ravel(), O.apply_normal(og, u[b]).ravel()) < 1e-11


def test_empty_batch_is_a_config_error(T):
    from paper_1705_07497_b200 import _lib
    og = O.Geometry(**GEOMS["ref_msp3"])
    op = T.make_direct_backend(pgeom(T, og))
    buf = cuda(np.zeros((og.n, og.n)), True)
    rc = _lib.lib().tomo_apply_normal(op._h, C.c_void_p(buf.data_ptr()), C.c_void_p(buf.data_ptr()), 0, None)
    assert rc == _lib.TOMO_ERR_CONFIG and b"batch" in _lib.lib().tomo_last_error()


def test_host_batches_are_streamed(T):
    """Host input + host output with several slices go through the chunked host<->device
    pipeline (tomo_capi.cu host_pipeline); results equal the device-resident path."""
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    rng = np.random.default_rng(21)
    for prec in ("f32", "f64"):
        f64 = prec == "f64"
        op = T.make_direct_backend(pgeom(T, og), precision=prec, max_batch=2)
        u = rng.standard_normal((7, og.n, og.n)) + 1j * rng.standard_normal((7, og.n, og.n))
        dev = cuda(u, True, f64)
        pinned = dev.cpu().pin_memory()
        for fn in (op.apply_normal, op.forward):
            want = fn(dev).cpu().numpy()
            got = fn(pinned)
            assert got.is_pinned() and np.array_equal(got.numpy(), want)
        s = op.forward(dev)
        assert np.array_equal(op.adjoint(s.cpu().pin_memory()).numpy(), op.adjoint(s).cpu().numpy())
        ur = dev.real.contiguous()
        assert np.array_equal(op.apply_normal_real(ur.cpu().pin_memory()).numpy(), op.apply_normal_real(ur).cpu().numpy())


def test_nccl_single_rank_plumbing(T):
    """The NCCL path of angle-block sharding (tomo_op_attach_nccl + the all-reduce after every
    adjoint, also inside the captured solver graphs) on a one-rank communicator: a shard's
    results equal the same shard with a no-op all-reduce hook."""
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    g = pgeom(T, og)
    blk = (0, og.n_angles // 2)
    hook = T.make_direct_backend(g, precision="f64", angle_block=blk)
    hook.set_allreduce(lambda *a: None)
    nccl = T.make_direct_backend(g, precision="f64", angle_block=blk)
    nccl.attach_nccl(T.nccl_unique_id(), 1, 0)
    rng = np.random.default_rng(31)
    u = cuda(rng.standard_normal((og.n, og.n)), False, True)
    assert np.array_equal(nccl.apply_normal_real(u).cpu().numpy(), hook.apply_normal_real(u).cpu().numpy())
    f = cuda(rng.standard_normal((og.n_angles // 2) * og.n_b) + 0j, True, True)
    a = nccl.chambolle_pock(f, alpha=1e-2, lambda_=1e-2, iters=2, cg_steps=3).cpu().numpy()
    b = hook.chambolle_pock(f, alpha=1e-2, lambda_=1e-2, iters=2, cg_steps=3).cpu().numpy()
    assert np.array_equal(a, b)
