"""GPU parity of the fused (Gram) backend: build_btb + apply_normal_fused
(proj/src/normal_ops.cpp:53-206) on the device, vs the fp64 oracle, the reference's own
golden vectors and the direct backend (direct and fused agree to 1e-10)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import cases, load, rel
from tests.test_gpu_parity import GEOMS, OP_TOL, OP_TOL_F64, PRECS, REC_TOL, cuda, gold_geom, pgeom

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(77)


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", list(GEOMS))
def test_fused_normal_vs_oracle(T, name, prec):
    f64 = prec == "f64"
    tol = OP_TOL_F64 if f64 else OP_TOL
    og = O.Geometry(**GEOMS[name])
    op = T.make_fused_backend(pgeom(T, og), precision=prec)
    info = op.info
    assert info.backend == 1
    assert info.gram_nnz == O.btb_nnz(og)  # same sparsity as build_btb's CSR
    n = og.n
    u = RNG.standard_normal((n, n)) + 1j * RNG.standard_normal((n, n))
    if not f64:
        u = u.astype(np.complex64)
    assert rel(op.apply_normal(cuda(u, True, f64)).cpu().numpy().ravel(), O.apply_normal_fused(og, u).ravel()) < tol
    ur = RNG.standard_normal((n, n))
    if not f64:
        ur = ur.astype(np.float32)
    ref = O.apply_normal_fused(og, ur.astype(np.complex128)).real
    assert rel(op.apply_normal_real(cuda(ur, False, f64)).cpu().numpy().ravel(), ref.ravel()) < tol


def test_fused_matches_direct_f64(T):
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    g = pgeom(T, og)
    n = og.n
    u = cuda(RNG.standard_normal((2, n, n)) + 1j * RNG.standard_normal((2, n, n)), True, True)
    a = T.make_fused_backend(g, precision="f64", max_batch=2).apply_normal(u).cpu().numpy()
    b = T.make_direct_backend(g, precision="f64", max_batch=2).apply_normal(u).cpu().numpy()
    assert rel(a, b) < 1e-10


GOLD = [c for c in cases() if "fused_normal_u" in load(c)]


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(c) for c in GOLD])
@pytest.mark.parametrize("prec", PRECS)
def test_fused_golden(T, path, prec):
    """vs apply_normal_fused / build_btb of the reference itself (tests/golden)."""
    gold = load(path)
    f64 = prec == "f64"
    op = T.make_fused_backend(gold_geom(T, gold), precision=prec)
    assert op.info.gram_nnz == int(gold["btb_nnz"])
    out = op.apply_normal(cuda(gold["u"], True, f64)).cpu().numpy().ravel()
    assert rel(out, gold["fused_normal_u"].ravel()) < (OP_TOL_F64 if f64 else OP_TOL)


def test_fused_batch_split_tasks(T):
    """window 13 -> Gram rows of up to 625 entries: every block is split into several warp
    tasks combined by the last-task ticket; batched slices must equal single ones."""
    og = O.Geometry(**GEOMS["ref_msp6"])
    op = T.make_fused_backend(pgeom(T, og), max_batch=3, precision="f64")
    n = og.n
    u = RNG.standard_normal((3, n, n)) + 1j * RNG.standard_normal((3, n, n))
    batched = op.apply_normal(cuda(u, True, True)).cpu().numpy()
    for b in range(3):
        assert rel(batched[b].ravel(), O.apply_normal_fused(og, u[b]).ravel()) < OP_TOL_F64
    again = op.apply_normal(cuda(u, True, True)).cpu().numpy()
    assert np.array_equal(again, batched)  # deterministic (fixed-order partial sums)


def test_fused_solvers_vs_oracle(T):
    og = O.Geometry(**GEOMS["ref_msp3"])
    n = og.n
    ph = O.random_ellipses(n, 8, 3)
    f, _ = O.synthesize(og, ph, 0.01, 3)
    op = T.make_fused_backend(pgeom(T, og), precision="f64")
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=5, cg_steps_per_update=5, update_tol_rel=0.0)
    mu, tr = op.split_bregman(cuda(f, True, True), cfg)
    ref, upd, _ = O.split_bregman(og, f, backend=1, alpha=10.0, lam=1.0, max_iters=5, cg_steps=5)
    assert rel(mu.cpu().numpy().ravel(), ref.ravel()) < REC_TOL
    rhs = RNG.standard_normal((n, n))
    x, st = op.cg(cuda(rhs, False, True), alpha=10.0, lambda_=1.0, steps=5)
    xr, _ = O.cg(og, O.system(backend=1, alpha=10.0, lam=1.0), rhs, steps=5)
    assert rel(x.cpu().numpy().ravel(), np.asarray(xr).ravel()) < 1e-8


def test_fused_angle_shards_sum_to_full(T):
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    g = pgeom(T, og)
    n = og.n
    u = cuda(RNG.standard_normal((n, n)), False, True)
    full = T.make_fused_backend(g, precision="f64").apply_normal_real(u).cpu().numpy()
    A = og.n_angles
    parts = []
    for a0, a1 in ((0, A // 3), (A // 3, A)):
        op = T.make_fused_backend(g, precision="f64", angle_block=(a0, a1))
        op.set_allreduce(lambda buf, count, stream: None)  # local partial only
        parts.append(op.apply_normal_real(u).cpu().numpy())
    assert rel(parts[0] + parts[1], full) < 1e-10


def test_fused_mem_cap(T):
    og = O.Geometry(**GEOMS["ref_msp3"])
    with pytest.raises(T.ConfigError, match="exceeds cap"):
        T.make_fused_backend(pgeom(T, og), mem_cap_bytes=1 << 10)
