"""The real-subspace (Hermitian half-grid) pipeline against the full-grid complex pipeline of the
same op: Re(N u) for a real image u through P1 on row pairs, m/2 + 1 grid rows, the mirrored W
gathers, the folded W^T and PB on row pairs equals the real part of the complex
apply of u + 0i (full grid, unfolded W^T) to rounding, for every FFT-pass variant (half-pruned
R = 2, R = 4, long rows with the persistent grid-row passes), batch shape (single slice,
slice groups on grid.y, lanes) and solver path."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(77)

GEOMS = {
    "n16_m32": dict(n=16, n_angles=10, win_lo=-2, win_hi=2),
    "msp3_n32": dict(n=32, n_angles=25, win_lo=-3, win_hi=3),
    "width6_n64": dict(n=64, n_angles=30, n_b=65, win_lo=-2, win_hi=3, tau=3 / 64 ** 2),
    "R4_n32": dict(n=32, n_angles=20, n_b=33, oversample=4, win_lo=-3, win_hi=3, tau=np.pi * 3 / (32 ** 2 * 4 * 3.5)),
    "n256_c1": dict(n=256, n_angles=60, n_b=367, win_lo=-2, win_hi=3, tau=3 / 256 ** 2),
    "n512_c2": dict(n=512, n_angles=90, n_b=725, win_lo=-3, win_hi=3, tau=3 / 512 ** 2),
    "n2048_m4096": dict(n=2048, n_angles=8, n_b=2049, win_lo=-2, win_hi=3, tau=3 / 2048 ** 2),
    "n1024_R4_m4096": dict(n=1024, n_angles=8, n_b=1025, oversample=4, win_lo=-2, win_hi=3,
                           tau=np.pi * 3 / (1024 ** 2 * 4 * 3.5)),
}


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def pgeom(T, og):
    return T.Geometry(n=og.n, n_angles=og.n_angles, n_b=og.n_b, oversample=og.oversample, win_lo=og.win_lo,
                      win_hi=og.win_hi, tau=og.tau)


def dev(x, complex_, f64):
    dt = (np.complex128 if complex_ else np.float64) if f64 else (np.complex64 if complex_ else np.float32)
    return torch.from_numpy(np.ascontiguousarray(x, dt)).cuda()


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("name", list(GEOMS))
def test_real_apply_equals_complex_apply(T, name, prec):
    f64 = prec == "f64"
    tol = 1e-13 if f64 else 3e-6
    og = O.Geometry(**GEOMS[name])
    op = T.make_direct_backend(pgeom(T, og), precision=prec)
    assert op.info.herm_tasks > 0, "the folded W^T was not built"
    if f64 and op.info.sym_tasks > 0:
        # mirror pairs (tests/test_gpu_sym.py): the secondaries take their primaries' weights, which
        # differ from their own by the rounding of the sample positions (|x| eps / h per weight)
        tol = 2e-11
    n = og.n
    for B in ((1, 3, 7) if n <= 512 else (1,)):
        u = RNG.standard_normal((B, n, n))
        real = op.apply_normal_real(dev(u, False, f64)).cpu().numpy().reshape(B, n, n)
        full = op.apply_normal(dev(u, True, f64)).cpu().numpy().reshape(B, n, n)
        err = rel(real, full.real)
        print(f"{name} {prec} B={B}: real vs Re(complex) rel-L2 {err:.2e}")
        assert err < tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("name", ["width6_n64", "R4_n32", "n512_c2"])
def test_backprojection_and_forward_of_real_image(T, name, prec):
    """Re(F_NU s) through the folded W^T vs the real part of the full adjoint; F_NU^* of a real
    image through the half grid vs the full forward of the same image as complex."""
    f64 = prec == "f64"
    tol = 1e-13 if f64 else 3e-6
    og = O.Geometry(**GEOMS[name])
    op = T.make_direct_backend(pgeom(T, og), precision=prec)
    s = RNG.standard_normal(og.P) + 1j * RNG.standard_normal(og.P)
    bp = op.backproject(dev(s, True, f64), weighted=False).cpu().numpy().ravel()
    adj = op.adjoint(dev(s, True, f64)).cpu().numpy().ravel()
    assert rel(bp, adj.real) < tol
    u = RNG.standard_normal((og.n, og.n))
    fr = op.forward_real(dev(u, False, f64)).cpu().numpy().ravel()
    fc = op.forward(dev(u, True, f64)).cpu().numpy().ravel()
    assert rel(fr, fc) < tol


@pytest.mark.parametrize("name", ["width6_n64", "R4_n32"])
def test_solvers_half_grid_vs_oracle(T, name):
    """CG and split Bregman (fp64, Chronopoulos-Gear, the half-grid path) vs the oracle."""
    og = O.Geometry(**GEOMS[name])
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    ph = O.random_ellipses(og.n, 10, 3)
    f, _ = O.synthesize(og, ph, 0.01, 3)
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=4, cg_steps_per_update=6, update_tol_rel=0.0)
    mu, _ = op.split_bregman(dev(f, True, True), cfg)
    mref, _, _ = O.split_bregman(og, f, backend=0, alpha=10.0, lam=1.0, max_iters=4, cg_steps=6)
    err = rel(mu.cpu().numpy().ravel(), mref.ravel())
    print(f"{name}: split Bregman 4x6 vs oracle {err:.2e}")
    assert err < 1e-6


_W_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1705_07497_b200 as T
from oracle import oracle as O
spec = eval(sys.argv[2]); prec = sys.argv[4]
og = O.Geometry(**spec)
op = T.make_direct_backend(T.Geometry(n=og.n, n_angles=og.n_angles, n_b=og.n_b, oversample=og.oversample,
                                      win_lo=og.win_lo, win_hi=og.win_hi, tau=og.tau), precision=prec)
rt, ct = (np.float64, np.complex128) if prec == "f64" else (np.float32, np.complex64)
rng = np.random.default_rng(5)
outs = []
for B in (1, 3, 7):
    u = rng.standard_normal((B, og.n, og.n))
    uc = u + 1j * rng.standard_normal((B, og.n, og.n))
    outs.append(op.forward_real(torch.from_numpy(u.astype(rt)).cuda()).cpu().numpy().ravel())
    outs.append(op.forward(torch.from_numpy(uc.astype(ct)).cuda()).cpu().numpy().ravel())
np.save(sys.argv[3], np.concatenate(outs))
"""


@pytest.mark.parametrize("prec", ["f32"])
@pytest.mark.parametrize("name", ["n16_m32", "width6_n64", "n256_c1", "n1024_R4_m4096"])
def test_w_vector_rows_bit_identical_to_scalar_gathers(T, name, prec, tmp_path):
    """fp32 width-6 W with 16-byte window-row loads (k_w_sep_v6, the default) vs the scalar gathers
    (TOMO_W_VEC=0): same arithmetic in the same order, bit-identical samples on the half grid
    (mirrored rows) and the full grid, single and batched launches, incl. edge-wrapping windows."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for vec in ("1", "0"):
        env = dict(os.environ, TOMO_AB="1", TOMO_W_VEC=vec)
        path = str(tmp_path / f"w{vec}.npy")
        subprocess.check_call([sys.executable, "-c", _W_CHILD, root, repr(GEOMS[name]), path, prec], env=env)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
