"""GPU operators from / to the reference's TOMOSPM1 files (load_or_build_sparse, bench.cpp:78-114;
save_sparse, sparse.cpp:68-106): Gram and surrogate T written by the reference itself are loaded
into device operators and checked against the oracle; the product's own files are compared with
the reference's bytes."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import tspm_util
from tests.golden_util import rel
from tests.test_gpu_parity import OP_TOL, OP_TOL_F64, PRECS, cuda, pgeom

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BTB = os.path.join(GOLD, "ref_btb_n16_a6_msp1.tspm")
T1 = os.path.join(GOLD, "ref_t_n16_a12_msp2_r1.tspm")
T2E = os.path.join(GOLD, "ref_t_n16_a12_msp2_r2e.tspm")
GB = O.Geometry(n=16, n_angles=6, win_lo=-1, win_hi=1)
G16 = O.Geometry(n=16, n_angles=12, win_lo=-2, win_hi=2)
RNG = np.random.default_rng(5)


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


@pytest.mark.parametrize("prec", PRECS)
def test_fused_from_reference_gram(T, prec):
    f64 = prec == "f64"
    op = T.NormalBackend(pgeom(T, GB), "fused", precision=prec, tspm=BTB)
    assert op.info.gram_nnz == tspm_util.read(BTB)["nnz"]
    u = RNG.standard_normal((16, 16)) + 1j * RNG.standard_normal((16, 16))
    if not f64:
        u = u.astype(np.complex64)
    out = op.apply_normal(cuda(u, True, f64)).cpu().numpy().ravel()
    assert rel(out, O.apply_normal_fused(GB, u).ravel()) < (OP_TOL_F64 if f64 else OP_TOL)


def test_saved_gram_is_the_reference_file(T, tmp_path):
    op = T.make_fused_backend(pgeom(T, GB), precision="f64")
    path = tmp_path / "btb.tspm"
    op.save_sparse(path, angle_subsample_d=1)
    mine, ref = tspm_util.read(path), tspm_util.read(BTB)
    for k in ("rows", "cols", "nnz", "symmetric", "n", "m_sp", "tau", "angle_count", "d", "r"):
        assert mine[k] == ref[k], k
    assert np.array_equal(mine["off"], ref["off"]) and np.array_equal(mine["col"], ref["col"])
    assert np.allclose(mine["val"], ref["val"], rtol=1e-13, atol=0)
    # fp64 host build: same sample order and product association as build_btb -> same bytes
    assert path.read_bytes() == open(BTB, "rb").read()


@pytest.mark.parametrize("path,r,eu", [(T1, 1, False), (T2E, 2, True)])
def test_surrogate_from_reference_t(T, path, r, eu):
    op = T.NormalBackend(pgeom(T, G16), "surrogate", precision="f64", tspm=path)
    assert op.info.surrogate_r == r
    st = tspm_util.stencil(tspm_util.read(path))
    assert np.allclose(op.stencil(), st, rtol=0, atol=0)
    u = RNG.standard_normal((16, 16))
    out = op.apply_normal_real(cuda(u, False, True)).cpu().numpy()
    assert rel(out, O.apply_stencil(16, r, st, u, euclidean=eu)) < 1e-12


@pytest.mark.parametrize("r,eu,ref", [(1, False, T1), (2, True, T2E)])
def test_saved_surrogate_matches_reference_t(T, tmp_path, r, eu, ref):
    op = T.make_surrogate_backend(pgeom(T, G16), radius_r=r, euclidean=eu, precision="f64")
    path = tmp_path / "t.tspm"
    op.save_sparse(path)
    mine, want = tspm_util.read(path), tspm_util.read(ref)
    assert np.array_equal(mine["off"], want["off"]) and np.array_equal(mine["col"], want["col"])
    assert (mine["n"], mine["r"], mine["tau"], mine["angle_count"]) == (want["n"], want["r"], want["tau"], want["angle_count"])
    assert np.allclose(mine["val"], want["val"], rtol=1e-10, atol=1e-14)
    back = T.NormalBackend(pgeom(T, G16), "surrogate", precision="f64", tspm=str(path))
    u = cuda(RNG.standard_normal((16, 16)), False, True)
    assert np.array_equal(back.apply_normal_real(u).cpu().numpy(), op.apply_normal_real(u).cpu().numpy())


def test_cache_metadata_mismatch(T):
    g = O.Geometry(n=16, n_angles=7, win_lo=-1, win_hi=1)
    with pytest.raises(T.ConfigError, match="metadata mismatch"):
        T.NormalBackend(pgeom(T, g), "fused", tspm=BTB)
    with pytest.raises(T.ConfigError):
        T.NormalBackend(pgeom(T, GB), "surrogate", tspm=BTB)  # a Gram is not a surrogate T
    with pytest.raises(T.ConfigError):
        T.NormalBackend(pgeom(T, GB), "direct", tspm=BTB)
