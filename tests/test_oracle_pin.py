"""Live pin: oracle restatement vs the reference's own code (oracle/_ref/libtomo_ref.so),
on cases beyond the committed golden vectors. Skipped where the reference build is absent
(e.g. on a GPU box without /root/reference and no prebuilt _ref)."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import refbind

pytestmark = pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.parametrize("n,A,msp", [(16, 7, 2), (24, 19, 3), (48, 37, 6), (64, 50, 12)])
def test_pin_operator(n, A, msp):
    ref = refbind.Ref(n, A, msp)
    g = O.Geometry(n=n, n_angles=A, win_lo=-msp, win_hi=msp)
    rng = np.random.default_rng(n * A)
    u = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    assert np.array_equal(O.points(g), ref.points())
    assert rel(O.apply_normal(g, u), ref.apply_normal(u)) < 1e-12
    s = rng.standard_normal(g.P) + 1j * rng.standard_normal(g.P)
    assert rel(O.type1(g, s), ref.type1(s)) < 1e-12


def test_pin_tau_override_and_sb():
    n, A, msp = 32, 21, 3
    tau = 2.5 / n ** 2
    ref = refbind.Ref(n, A, msp, tau)
    g = O.Geometry(n=n, n_angles=A, win_lo=-msp, win_hi=msp, tau=tau)
    ph = refbind.shepp_logan(n)
    assert np.array_equal(ph, O.shepp_logan(n))
    f = ref.synthesize(ph, 0.5, 3)
    mu_r, upd_r, _, _ = ref.split_bregman(f, backend=0, alpha=3.0, lam=2.0, iters=4, cg_steps=6)
    mu_o, upd_o, _ = O.split_bregman(g, f, backend=0, alpha=3.0, lam=2.0, max_iters=4, cg_steps=6)
    # Shrink thresholds amplify last-bit FFT differences (1e-13 after one outer iteration,
    # ~1e-6 after four); the product bar is 1e-3.
    assert rel(mu_o, mu_r) < 1e-5


@pytest.mark.parametrize("backend", [0, 2])
def test_split_bregman_data_feedback_pinned(backend):
    """SolverConfig::data_feedback (solver.cpp:176-187, 283-286): outer residual feedback on the
    data term, and for the surrogate the feedback contraction floor sigma; oracle vs reference."""
    if not refbind.available():
        pytest.skip("oracle/_ref not built")
    n, A, msp = 32, 25, 3
    ref = refbind.Ref(n, A, msp)
    g = O.Geometry(n=n, n_angles=A, win_lo=-msp, win_hi=msp, tau=ref.tau)
    ph = refbind.shepp_logan(n)
    f = ref.synthesize(ph, 0.0, 0)
    mu_r, upd_r, sg_r, _ = ref.split_bregman(f, backend=backend, r=1, alpha=10.0 if backend == 0 else 1.0,
                                             lam=1.0, iters=4, cg_steps=4, feedback=True)
    mu_o, upd_o, tr = O.split_bregman(g, f, backend=backend, r=1, alpha=10.0 if backend == 0 else 1.0, lam=1.0,
                                      max_iters=4, cg_steps=4, feedback=True)
    assert abs(tr.sigma - sg_r) <= 1e-6 * max(abs(sg_r), 1.0)
    assert np.linalg.norm(mu_o - mu_r) / np.linalg.norm(mu_r) < 1e-6
    assert np.allclose(upd_o, upd_r, rtol=1e-6)
    # feedback changes the iterates (it is not a no-op)
    mu_n, _, _ = O.split_bregman(g, f, backend=backend, r=1, alpha=10.0 if backend == 0 else 1.0, lam=1.0,
                                 max_iters=4, cg_steps=4)
    assert np.linalg.norm(mu_n - mu_o) > 1e-6 * np.linalg.norm(mu_o)
