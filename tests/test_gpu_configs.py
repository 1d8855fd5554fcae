"""Oracle parity at the five BASELINE.json configs (c1-c5), on the exact geometries, precisions,
batch shapes and solver settings `bench.py` times (its CONFIGS table is imported, so the kernel
instantiations here are the benched ones).

Inputs are synthesised once on the host by the oracle (seeded random ellipses + 1 % complex
Gaussian noise, `orc_synthesize`), and the same bytes go to the CUDA path (through the C ABI)
and to the fp64 CPU oracle. Tolerances (north star): rel-L2 <= 1e-5 for one fp32 operator
application, <= 1e-3 for reconstructions after a fixed iteration count; the fp64 applies are
held to 1e-10. Each measured rel-L2 is printed and, when TOMO_PARITY_LOG names a file, appended
to it as one JSON line.

Reference semantics checked (paths under /root/reference):
  c1  apply_normal_real (proj/src/normal_ops.cpp:333-340) x 20 per call, then cg_solve on the
      Tikhonov system (proj/src/solver.cpp:56-95, 309-337; D11: 20 fixed steps)
  c2  split_bregman_tv (proj/src/solver.cpp:219-307), 50 outer x 10 CG, m_sp = 3 window
  c3  apply_normal complex (proj/src/normal_ops.cpp:321-331), calls of 3 inputs
  c4  split_bregman_tv on the surrogate backend (build_surrogate, normal_ops.cpp:232-283),
      30 outer x 5 CG, several slices per call
  c5  Chambolle-Pock (extension D10) at R = 4, one outer iteration x 15 CG
"""
import json
import os
import time

import numpy as np
import pytest

import bench
from oracle import oracle as O
from tests.golden_util import rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OP_TOL = 1e-5       # north star: one fp32 operator application
OP_TOL_F64 = 1e-10  # fp64 operator vs the fp64 oracle: rounding only
REC_TOL = 1e-3      # north star: reconstructions after a fixed iteration count


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def record(config, what, err, tol, **extra):
    line = {"config": config, "check": what, "rel_l2": err, "tol": tol, **extra}
    print(json.dumps(line), flush=True)
    path = os.environ.get("TOMO_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(line) + "\n")
    assert err <= tol, line


def geoms(T, c):
    """The bench's geometry (bench.make_geom) and the same geometry for the oracle."""
    g = bench.make_geom(T, c)
    og = O.Geometry(n=g.n, n_angles=g.n_angles, n_b=g.n_b, oversample=g.oversample, win_lo=g.win_lo,
                    win_hi=g.win_hi, tau=g.tau)
    return g, og


def synth(og, seed):
    ph = O.random_ellipses(og.n, 10, seed)
    f, _ = O.synthesize(og, ph, 0.01, seed)
    return ph, f


def dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x, dtype)).cuda()


def test_c1_applies_and_tikhonov(T):
    c = bench.CONFIGS["c1"]
    g, og = geoms(T, c)
    B = c["batch"]  # 20 inputs per call: three lanes of 7/7/6 slices (W / W^T slice groups on grid.y)
    op = T.make_direct_backend(g, precision=c["prec"], max_batch=B)
    ph, f = synth(og, 3000)
    rng = np.random.default_rng(11)
    u = np.stack([ph] + [rng.standard_normal((og.n, og.n)) for _ in range(B - 1)])
    out = op.apply_normal_real(dev(u, np.float64)).cpu().numpy()
    errs = [rel(out[b], O.apply_normal_real(og, u[b])) for b in range(B)]
    record("c1", f"apply_normal_real x{B} (worst)", max(errs), OP_TOL_F64, batch=B)
    mu = op.tikhonov(dev(f, np.complex128), alpha=c["alpha"], steps=c["cg"]).cpu().numpy()
    ref = O.tikhonov_identity(og, f, alpha=c["alpha"], steps=c["cg"])
    record("c1", f"tikhonov {c['cg']} CG", rel(mu, ref), REC_TOL)


def test_c2_split_bregman(T):
    c = bench.CONFIGS["c2"]
    g, og = geoms(T, c)
    assert (g.win_lo, g.win_hi) == (-3, 3), "c2 runs the reference's m_sp = 3 window"
    op = T.make_direct_backend(g, precision=c["prec"])
    _, f = synth(og, 1000)
    cfg = T.SolverConfig(alpha=c["alpha"], lambda_=c["lam"], max_bregman_iters=c["iters"],
                         cg_steps_per_update=c["cg"], update_tol_rel=0.0)
    mu, tr = op.split_bregman(dev(f, np.complex128), cfg)
    t0 = time.perf_counter()
    ref, upd, otr = O.split_bregman(og, f, backend=0, alpha=c["alpha"], lam=c["lam"], max_iters=c["iters"],
                                    cg_steps=c["cg"])
    t_oracle = time.perf_counter() - t0
    assert tr[0].iterations == otr.iterations == c["iters"]
    record("c2", f"split_bregman {c['iters']}x{c['cg']}", rel(mu.cpu().numpy(), ref), REC_TOL,
           oracle_s=round(t_oracle, 1))
    record("c2", "update_l1 trace", rel(tr[0].update_l1, upd), REC_TOL)


def test_c2_width6_window(T):
    """The width-6 [-2, 3] window (BASELINE c1/c3's "kernel width 6") on the c2 geometry: the
    6-tap kernel instantiations at m = 1024 in fp64, through a shorter split Bregman."""
    c = dict(bench.CONFIGS["c2"], lo=-2, hi=3)
    g, og = geoms(T, c)
    op = T.make_direct_backend(g, precision="f64")
    _, f = synth(og, 1001)
    cfg = T.SolverConfig(alpha=c["alpha"], lambda_=c["lam"], max_bregman_iters=10, cg_steps_per_update=c["cg"],
                         update_tol_rel=0.0)
    mu, _ = op.split_bregman(dev(f, np.complex128), cfg)
    ref, _, _ = O.split_bregman(og, f, backend=0, alpha=c["alpha"], lam=c["lam"], max_iters=10, cg_steps=c["cg"])
    record("c2[-2,3]", "split_bregman 10x10", rel(mu.cpu().numpy(), ref), REC_TOL)


def test_c3_complex_applies(T):
    c = bench.CONFIGS["c3"]
    g, og = geoms(T, c)
    B = c["batch"]  # calls of 3 independent inputs on three lanes
    op = T.make_direct_backend(g, precision=c["prec"], max_batch=B)
    rng = np.random.default_rng(7)
    u = (rng.standard_normal((B, og.n, og.n)) + 1j * rng.standard_normal((B, og.n, og.n))).astype(np.complex64)
    out = op.apply_normal(dev(u, np.complex64)).cpu().numpy()
    errs = [rel(out[b], O.apply_normal(og, u[b])) for b in range(B)]
    record("c3", f"apply_normal complex64 x{B} (worst)", max(errs), OP_TOL, batch=B)
    # one input per call (the reference's time_apply shape)
    out1 = op.apply_normal(dev(u[:1], np.complex64)).cpu().numpy()
    record("c3", "apply_normal complex64 x1", rel(out1[0], O.apply_normal(og, u[0])), OP_TOL)


def test_c4_surrogate_batch(T):
    c = bench.CONFIGS["c4"]
    g, og = geoms(T, c)
    B = 4
    op = T.make_surrogate_backend(g, radius_r=c["r"], max_batch=B)
    fs = [synth(og, 2000 + s)[1] for s in range(B)]
    cfg = T.SolverConfig(alpha=c["alpha"], lambda_=c["lam"], max_bregman_iters=c["iters"],
                         cg_steps_per_update=c["cg"], update_tol_rel=0.0)
    mu, tr = op.split_bregman(dev(np.stack(fs), np.complex64), cfg)
    mu = mu.cpu().numpy()
    sig = O.surrogate_sigma(og, c["r"], c["alpha"], c["lam"])
    record("c4", "sigma (Lanczos)", abs(tr[0].stabilization_shift - sig) / max(abs(sig), 1e-30), REC_TOL)
    errs = []
    for b in range(B):
        ref, _, _ = O.split_bregman(og, fs[b], backend=2, r=c["r"], alpha=c["alpha"], lam=c["lam"],
                                    max_iters=c["iters"], cg_steps=c["cg"])
        errs.append(rel(mu[b], ref))
    record("c4", f"surrogate split_bregman {c['iters']}x{c['cg']} x{B} slices (worst)", max(errs), REC_TOL)


def test_c5_apply_and_chambolle_pock(T):
    c = bench.CONFIGS["c5"]
    g, og = geoms(T, c)
    assert og.oversample == 4 and og.m == 8192
    op = T.make_direct_backend(g, precision=c["prec"])
    ph, f = synth(og, 5000)
    out = op.apply_normal_real(dev(ph, np.float64)).cpu().numpy()
    record("c5", "apply_normal_real f64", rel(out, O.apply_normal_real(og, ph)), OP_TOL_F64)
    cp = dict(alpha=c["alpha"], tau_cp=c["tau_cp"], sigma_cp=c["sigma_cp"], theta=c["theta"], iters=1)
    fd = dev(f, np.complex128)
    # (a) one CP iteration with a 10-step prox CG: before CG's transient (below), GPU and oracle
    #     agree to rounding
    mu = op.chambolle_pock(fd, lambda_=c["lam"], cg_steps=10, **cp).cpu().numpy()
    ref = O.chambolle_pock(og, f, lam=c["lam"], cg_steps=10, **cp)
    record("c5", "chambolle_pock 1x10 CG", rel(mu, ref), REC_TOL)
    # (b) the config's 1 x 15: the prox system I + tau*alpha*N has kappa ~ 7e5 here, and between
    #     CG steps 13 and 15 its Ritz values converge and CG amplifies per-apply rounding to the
    #     1e-4 level (the GPU's two CG forms differ by 1.4e-4 from each other); DESIGN.md §5. The
    #     bound is 1e-3 or, if larger, 3x the oracle's own spread when each of its applies is
    #     perturbed at the rounding level of an equally exact implementation (1e-16 relative).
    mu = op.chambolle_pock(fd, lambda_=c["lam"], cg_steps=c["cg"], **cp).cpu().numpy()
    t0 = time.perf_counter()
    ref = O.chambolle_pock(og, f, lam=c["lam"], cg_steps=c["cg"], **cp)
    t_oracle = time.perf_counter() - t0
    try:
        O.set_perturbation(1e-16, seed=3)
        ref_p = O.chambolle_pock(og, f, lam=c["lam"], cg_steps=c["cg"], **cp)
    finally:
        O.set_perturbation(0.0)
    spread = rel(ref_p, ref)
    record("c5", f"chambolle_pock 1x{c['cg']} CG (bound: 3 x oracle rounding spread)", rel(mu, ref),
           max(REC_TOL, 3.0 * spread), oracle_rounding_spread=spread, oracle_s=round(t_oracle, 1))
