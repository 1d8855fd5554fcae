"""Oracle restatement vs golden vectors produced by the reference itself
(tests/golden/make_golden.py; the reference sources built against the Eigen-API shim)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import cases, load, rel

CASES = cases()


def geom(d):
    msp = int(d["m_sp"])
    return O.Geometry(n=int(d["n"]), n_angles=int(d["n_angles"]), win_lo=-msp, win_hi=msp,
                      tau=float(d["tau"]))


@pytest.fixture(params=CASES, ids=[os.path.basename(c) for c in CASES])
def gold(request):
    return load(request.param)


def test_golden_present():
    assert len(CASES) >= 3


def test_points_and_plan_bit_exact(gold):
    g = geom(gold)
    assert np.array_equal(O.points(g), gold["points"])
    near, e1, e2, e3 = O.plan(g)
    assert np.array_equal(near, gold["nearest"])
    assert np.array_equal(e1, gold["e1"]) and np.array_equal(e2, gold["e2"])
    assert np.array_equal(e3, gold["e3"])


def test_type2_type1(gold):
    g = geom(gold)
    assert rel(O.type2(g, gold["u"]), gold["type2_u"]) < 1e-13
    assert rel(O.type1(g, gold["s"]), gold["type1_s"]) < 1e-13


def test_normal_ops(gold):
    g = geom(gold)
    assert rel(O.apply_normal(g, gold["u"]), gold["normal_u"]) < 1e-13
    assert rel(O.apply_normal_real(g, gold["ur"]), gold["normal_real_ur"]) < 1e-13
    if "fused_normal_u" in gold:
        assert rel(O.apply_normal_fused(g, gold["u"]), gold["fused_normal_u"]) < 1e-13
        assert O.btb_nnz(g) == int(gold["btb_nnz"])


def test_surrogate(gold):
    g = geom(gold)
    n = g.n
    for r in (1, 2):
        st = O.surrogate_stencil(g, r)
        assert rel(st, gold[f"stencil_r{r}"]) < 1e-12
        assert rel(O.apply_stencil(n, r, st, gold["ur"]), gold[f"surrogate_ur_r{r}"]) < 1e-12


def test_synthesize_bit_compatible(gold):
    g = geom(gold)
    f, sigma = O.synthesize(g, gold["phantom"], 0.01, 9)
    assert abs(sigma - float(gold["noise_sigma"])) <= 1e-12 * sigma
    assert rel(f, gold["data"]) < 1e-13


def test_cg_and_solvers(gold):
    g = geom(gold)
    x, st = O.cg(g, O.system(0, alpha=10.0, lam=1.0), gold["cg_rhs"], steps=5)
    assert rel(x, gold["cg_x"]) < 1e-9
    assert abs(st.min_ritz - float(gold["cg_min_ritz"])) <= 1e-9 * abs(float(gold["cg_min_ritz"]))
    mu, upd, tr = O.split_bregman(g, gold["data"], backend=0, alpha=10.0, lam=1.0, max_iters=5, cg_steps=5)
    assert rel(mu, gold["sb_direct_mu"]) < 1e-6  # shrink is non-smooth: reduction order shows at 1e-8
    assert rel(upd, gold["sb_direct_upd"]) < 1e-6
    assert abs(tr.imag_leakage - float(gold["sb_direct_leak"])) < 1e-12
    mu, upd, tr = O.split_bregman(g, gold["data"], backend=2, r=1, alpha=1.0, lam=1.0, max_iters=5, cg_steps=5)
    assert abs(tr.sigma - float(gold["sb_sur_sigma"])) <= 1e-8 * abs(float(gold["sb_sur_sigma"])) + 1e-12
    assert rel(mu, gold["sb_sur_mu"]) < 1e-6
    mu = O.tikhonov_identity(g, gold["data"], alpha=1.0, steps=20)
    # 20 CG steps amplify the reduction order: the reference build's sequential sums (the Eigen
    # shim) vs the oracle's compensated inner products differ by 1.5e-7 at n = 32, m_sp = 3
    assert rel(mu, gold["tikhonov_mu"]) < 1e-6
