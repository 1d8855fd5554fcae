"""Mirror pairs of the parallel-beam samples: with a window [1 - hi, hi] the bins
t and 2 (n_b / 2) - t of one angle have mirror-image interpolation windows, so for real images the
normal operator runs W on one sample per pair and the folded W^T of the pairs' primaries; with the
reference's symmetric window [-m_sp, m_sp] the partner's window is shifted by one node and the fold
reads pair sums inside the common window ("overlap pairs"). Checked
against the same op built without the pairs (TOMO_AB=1 TOMO_SYM=0: the full folded W^T and the full
W) and against the fp64 oracle, for single slices, slice groups and the solvers."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(505)

GEOMS = {
    "width6_n64": dict(n=64, n_angles=30, n_b=65, win_lo=-2, win_hi=3, tau=3 / 64 ** 2),
    "width6_even_nb": dict(n=64, n_angles=24, n_b=92, win_lo=-2, win_hi=3, tau=3 / 64 ** 2),
    "width4_n32": dict(n=32, n_angles=17, n_b=47, win_lo=-1, win_hi=2, tau=3 / 32 ** 2),
    "R4_n64": dict(n=64, n_angles=20, n_b=91, oversample=4, win_lo=-2, win_hi=3, tau=np.pi * 3 / (64 ** 2 * 4 * 3.5)),
    "n256_c1": dict(n=256, n_angles=60, n_b=367, win_lo=-2, win_hi=3, tau=3 / 256 ** 2),
}
# symmetric windows [-m_sp, m_sp] around floor(x / h) (the reference's): the partner's window is the
# mirror image shifted by one node -> "overlap pairs" (W whole, pair sums, 62/98 of the fold at m_sp = 3)
OVERLAP = {
    "msp3_n32": dict(n=32, n_angles=25, win_lo=-3, win_hi=3),
    "msp3_n64": dict(n=64, n_angles=30, n_b=91, win_lo=-3, win_hi=3, tau=3 / 64 ** 2),
    "msp2_n64": dict(n=64, n_angles=30, n_b=65, win_lo=-2, win_hi=2, tau=3 / 64 ** 2),
    "msp3_even_nb": dict(n=64, n_angles=24, n_b=92, win_lo=-3, win_hi=3, tau=3 / 64 ** 2),
    "R4_msp3_n32": dict(n=32, n_angles=20, n_b=33, oversample=4, win_lo=-3, win_hi=3,
                        tau=np.pi * 3 / (32 ** 2 * 4 * 3.5)),
    "n128_c2_like": dict(n=128, n_angles=45, n_b=181, win_lo=-3, win_hi=3, tau=3 / 128 ** 2),
    # neither symmetric nor its own mirror image: common window [-1, 2], plain W + pair-sum pass
    "asym_m1p3": dict(n=64, n_angles=26, n_b=77, win_lo=-1, win_hi=3, tau=3 / 64 ** 2),
}


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def pgeom(T, og):
    return T.Geometry(n=og.n, n_angles=og.n_angles, n_b=og.n_b, oversample=og.oversample, win_lo=og.win_lo,
                      win_hi=og.win_hi, tau=og.tau)


def make_ops(T, og, prec):
    """(op with the mirror pairs, the same op without them)."""
    op = T.make_direct_backend(pgeom(T, og), precision=prec, max_batch=8)
    os.environ["TOMO_AB"], os.environ["TOMO_SYM"] = "1", "0"
    try:
        ref = T.make_direct_backend(pgeom(T, og), precision=prec, max_batch=8)
    finally:
        del os.environ["TOMO_SYM"], os.environ["TOMO_AB"]
    return op, ref


def dev(x, f64):
    return torch.from_numpy(np.ascontiguousarray(x, np.float64 if f64 else np.float32)).cuda()


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("name", list(GEOMS))
def test_pairs_found_and_apply_matches(T, name, prec):
    f64 = prec == "f64"
    og = O.Geometry(**GEOMS[name])
    op, ref = make_ops(T, og, prec)
    inf, rinf = op.info, ref.info
    assert rinf.sym_tasks == 0 and inf.sym_tasks > 0
    # nearly every sample is paired (not: the zero frequency, bins without a mirror bin, samples on
    # a grid line), so W runs on about half of them and the fold keeps about half its entries
    assert inf.sym_pairs > 0.8 * inf.P and inf.sym_pairs % 2 == 0
    assert inf.sym_P == inf.P - inf.sym_pairs // 2
    assert inf.sym_nnz < 0.62 * inf.herm_nnz
    n = og.n
    for B in (1, 3, 7):
        u = RNG.standard_normal((B, n, n))
        a = op.apply_normal_real(dev(u, f64)).cpu().numpy().reshape(B, n, n)
        b = ref.apply_normal_real(dev(u, f64)).cpu().numpy().reshape(B, n, n)
        err = rel(a, b)
        print(f"{name} {prec} B={B}: pairs vs full fold rel-L2 {err:.2e} "
              f"(P {inf.P} -> {inf.sym_P}, fold nnz {inf.herm_nnz} -> {inf.sym_nnz})")
        assert err < (2e-11 if f64 else 3e-6)
    if f64:
        u = RNG.standard_normal((n, n))
        want = O.apply_normal_real(og, u)
        got = op.apply_normal_real(dev(u, True)).cpu().numpy().reshape(n, n)
        err = rel(got, want)
        print(f"{name}: pairs vs oracle rel-L2 {err:.2e}")
        assert err < 1e-10


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("name", list(OVERLAP))
def test_overlap_pairs_apply_matches(T, name, prec):
    f64 = prec == "f64"
    og = O.Geometry(**OVERLAP[name])
    op, ref = make_ops(T, og, prec)
    inf, rinf = op.info, ref.info
    assert rinf.sym_tasks == 0 and inf.sym_tasks > 0 and inf.herm_tasks > 0
    assert inf.sym_pairs > 0.8 * inf.P and inf.sym_P == inf.P  # W stays whole
    assert inf.sym_nnz < 0.72 * inf.herm_nnz
    n = og.n
    for B in (1, 3, 7):
        u = RNG.standard_normal((B, n, n))
        a = op.apply_normal_real(dev(u, f64)).cpu().numpy().reshape(B, n, n)
        b = ref.apply_normal_real(dev(u, f64)).cpu().numpy().reshape(B, n, n)
        err = rel(a, b)
        print(f"{name} {prec} B={B}: overlap pairs vs full fold rel-L2 {err:.2e} "
              f"(fold nnz {inf.herm_nnz} -> {inf.sym_nnz})")
        assert err < (2e-11 if f64 else 3e-6)
    if f64:
        u = RNG.standard_normal((n, n))
        got = op.apply_normal_real(dev(u, True)).cpu().numpy().reshape(n, n)
        err = rel(got, O.apply_normal_real(og, u))
        print(f"{name}: overlap pairs vs oracle rel-L2 {err:.2e}")
        assert err < 1e-10


@pytest.mark.parametrize("name", ["msp3_n64", "R4_msp3_n32"])
def test_pair_sum_pass_matches_unit_w(T, name):
    """The fallback of wide (w > 7) windows — the plain W followed by the pair-sum pass
    (TOMO_AB=1 TOMO_PAIR_W=0) — against the default W by mirror-pair units: the same operator."""
    og = O.Geometry(**OVERLAP[name])
    op = T.make_direct_backend(pgeom(T, og), precision="f64", max_batch=8)
    os.environ["TOMO_AB"], os.environ["TOMO_PAIR_W"] = "1", "0"
    try:
        alt = T.make_direct_backend(pgeom(T, og), precision="f64", max_batch=8)
    finally:
        del os.environ["TOMO_PAIR_W"], os.environ["TOMO_AB"]
    assert alt.info.sym_tasks == op.info.sym_tasks > 0
    n = og.n
    for B in (1, 5):
        u = RNG.standard_normal((B, n, n))
        a = op.apply_normal_real(dev(u, True)).cpu().numpy()
        b = alt.apply_normal_real(dev(u, True)).cpu().numpy()
        print(f"{name} B={B}: unit W vs W + pair-sum pass rel-L2 {rel(a, b):.2e}")
        assert rel(a, b) < 2e-11


def test_wide_symmetric_window_uses_the_pass(T):
    """m_sp = 6 (13-node windows): no unit W (union window > 8 nodes), the pass runs; vs the oracle."""
    og = O.Geometry(n=32, n_angles=20, n_b=47, win_lo=-6, win_hi=6)
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    assert op.info.sym_tasks > 0
    u = RNG.standard_normal((og.n, og.n))
    got = op.apply_normal_real(dev(u, True)).cpu().numpy().reshape(og.n, og.n)
    assert rel(got, O.apply_normal_real(og, u)) < 1e-10


def test_operator_is_symmetric(T):
    """<N u, v> = <u, N v>: the mirror-pair operator is U^T U of one interpolation U; the overlap-pair
    operator is symmetric to the rounding of the sample positions."""
    _operator_is_symmetric(T, GEOMS["width6_n64"], 1e-13)
    _operator_is_symmetric(T, OVERLAP["msp3_n64"], 1e-11)


def _operator_is_symmetric(T, geom, tol):
    og = O.Geometry(**geom)
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    n = og.n
    u, v = RNG.standard_normal((n, n)), RNG.standard_normal((n, n))
    nu = op.apply_normal_real(dev(u, True)).cpu().numpy().ravel()
    nv = op.apply_normal_real(dev(v, True)).cpu().numpy().ravel()
    a, b = float(nu @ v.ravel()), float(nv @ u.ravel())
    assert abs(a - b) <= tol * max(abs(a), abs(b))
    assert float(nu @ u.ravel()) > 0


@pytest.mark.parametrize("name", ["width6_n64", "R4_n64", "msp3_n64"])
def test_solvers_match_full_fold(T, name):
    og = O.Geometry(**{**GEOMS, **OVERLAP}[name])
    op, ref = make_ops(T, og, "f64")
    ph = O.random_ellipses(og.n, 10, 3)
    f, _ = O.synthesize(og, ph, 0.01, 3)
    fd = torch.from_numpy(f).cuda()
    a = op.tikhonov(fd, alpha=1.0, steps=12).cpu().numpy().ravel()
    b = ref.tikhonov(fd, alpha=1.0, steps=12).cpu().numpy().ravel()
    want = O.tikhonov_identity(og, f, alpha=1.0, steps=12)
    print(f"{name}: tikhonov pairs vs full {rel(a, b):.2e}, vs oracle {rel(a, want.ravel()):.2e}")
    # the pair operator differs from W^T W by ~2e-14 (the rounding of the sample positions); the
    # Tikhonov system's condition number (~5e6 at alpha = 1) scales that into the iterates
    assert rel(a, b) < 1e-6 and rel(a, want.ravel()) < 1e-6
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=4, cg_steps_per_update=6, update_tol_rel=0.0)
    ma, _ = op.split_bregman(fd, cfg)
    mb, _ = ref.split_bregman(fd, cfg)
    mo, _, _ = O.split_bregman(og, f, backend=0, alpha=10.0, lam=1.0, max_iters=4, cg_steps=6)
    ea, eo = rel(ma.cpu().numpy().ravel(), mb.cpu().numpy().ravel()), rel(ma.cpu().numpy().ravel(), mo.ravel())
    print(f"{name}: split Bregman pairs vs full {ea:.2e}, vs oracle {eo:.2e}")
    assert ea < 1e-6 and eo < 1e-3
