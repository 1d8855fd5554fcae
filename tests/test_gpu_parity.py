"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle and the reference's own
golden vectors. Tolerances are the north star's: rel-L2 <= 1e-5 for one fp32 operator
application, <= 1e-3 for reconstructions after a fixed iteration count."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import cases, load, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OP_TOL = 1e-5    # north star: one fp32 operator application
REC_TOL = 1e-3   # north star: reconstructions after a fixed iteration count


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def pgeom(T, og: O.Geometry):
    return T.Geometry(n=og.n, n_angles=og.n_angles, n_b=og.n_b, oversample=og.oversample, win_lo=og.win_lo,
                      win_hi=og.win_hi, tau=og.tau)


def cuda(x, complex_=False, f64=False):
    if f64:
        dt = np.complex128 if complex_ else np.float64
    else:
        dt = np.complex64 if complex_ else np.float32
    return torch.from_numpy(np.ascontiguousarray(x, dt)).cuda()


# fp32 operator parity is the north star's 1e-5; the fp64 path (used by the W-backend
# solvers) must agree with the fp64 oracle to rounding.
OP_TOL_F64 = 1e-11
PRECS = ["f32", "f64"]


RNG = np.random.default_rng(2024)

GEOMS = {
    "ref_msp6": dict(n=32, n_angles=25, win_lo=-6, win_hi=6),
    "ref_msp3": dict(n=32, n_angles=25, win_lo=-3, win_hi=3),
    "ref_msp12": dict(n=32, n_angles=25, win_lo=-12, win_hi=12),  # digits12: 25 taps (wide W kernel)
    "width6_odd_nb": dict(n=64, n_angles=30, n_b=65, win_lo=-2, win_hi=3, tau=3 / 64 ** 2),
    "R4_gl_tau": dict(n=32, n_angles=20, n_b=33, oversample=4, win_lo=-3, win_hi=3,
                      tau=np.pi * 3 / (32 ** 2 * 4 * 3.5)),
    "n16_m32": dict(n=16, n_angles=10, win_lo=-2, win_hi=2),  # smallest grid (m = 32)
    "n128": dict(n=128, n_angles=50, n_b=129, win_lo=-2, win_hi=3, tau=3 / 128 ** 2),
}

# Long rows (m = 4096): the persistent FFT-pass kernels (m >= 4096), the split twiddle reads, and
# at R = 2 the quarter-pruned pass variants; few angles keep the oracle's W/W^T cheap.
LARGE_GEOMS = {
    "n2048_m4096": dict(n=2048, n_angles=8, n_b=2049, win_lo=-2, win_hi=3, tau=3 / 2048 ** 2),
    "n1024_R4_m4096": dict(n=1024, n_angles=8, n_b=1025, oversample=4, win_lo=-2, win_hi=3,
                           tau=np.pi * 3 / (1024 ** 2 * 4 * 3.5)),
    # m = 8192 (c5's grid): fp64 grid rows split over two CTAs (k_t2_cols_dif / k_t1_cols_dif)
    "n2048_R4_m8192": dict(n=2048, n_angles=4, n_b=2049, oversample=4, win_lo=-2, win_hi=3,
                           tau=np.pi * 3 / (2048 ** 2 * 4 * 3.5)),
}


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("rows", [3, 600])
@pytest.mark.parametrize("m", [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192])
def test_fft_rows(T, m, prec, rows):
    f64 = prec == "f64"
    tol = 1e-13 if f64 else 2e-6
    rows = min(rows, max(3, (1 << 23) // m))
    x = RNG.standard_normal((rows, m)) + 1j * RNG.standard_normal((rows, m))
    out = T.tomo.fft_rows(cuda(x, True, f64)).cpu().numpy()
    assert rel(out, np.fft.fft(x, axis=1)) < tol
    outi = T.tomo.fft_rows(cuda(x, True, f64), inverse=True).cpu().numpy()
    assert rel(outi, np.fft.ifft(x, axis=1) * m) < tol


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", list(GEOMS))
def test_forward_adjoint_normal(T, name, prec):
    f64 = prec == "f64"
    tol = OP_TOL_F64 if f64 else OP_TOL
    og = O.Geometry(**GEOMS[name])
    op = T.make_direct_backend(pgeom(T, og), precision=prec)
    n = og.n
    u = RNG.standard_normal((n, n)) + 1j * RNG.standard_normal((n, n))
    s = RNG.standard_normal(og.P) + 1j * RNG.standard_normal(og.P)
    if not f64:  # same input bytes to both sides
        u = u.astype(np.complex64)
        s = s.astype(np.complex64)
    assert rel(op.forward(cuda(u, True, f64)).cpu().numpy().ravel(), O.type2(og, u)) < tol
    assert rel(op.adjoint(cuda(s, True, f64)).cpu().numpy().ravel(), O.type1(og, s).ravel()) < tol
    assert rel(op.apply_normal(cuda(u, True, f64)).cpu().numpy().ravel(), O.apply_normal(og, u).ravel()) < tol
    ur = RNG.standard_normal((n, n))
    if not f64:
        ur = ur.astype(np.float32)
    assert rel(op.apply_normal_real(cuda(ur, False, f64)).cpu().numpy().ravel(), O.apply_normal_real(og, ur).ravel()) < tol


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", list(LARGE_GEOMS))
def test_long_rows_vs_oracle(T, name, prec):
    f64 = prec == "f64"
    tol = OP_TOL_F64 if f64 else OP_TOL
    og = O.Geometry(**LARGE_GEOMS[name])
    op = T.make_direct_backend(pgeom(T, og), precision=prec)
    n = og.n
    u = RNG.standard_normal((n, n)) + 1j * RNG.standard_normal((n, n))
    ur = RNG.standard_normal((n, n))
    if not f64:
        u = u.astype(np.complex64)
        ur = ur.astype(np.float32)
    assert rel(op.apply_normal(cuda(u, True, f64)).cpu().numpy().ravel(), O.apply_normal(og, u).ravel()) < tol
    assert rel(op.apply_normal_real(cuda(ur, False, f64)).cpu().numpy().ravel(), O.apply_normal_real(og, ur).ravel()) < tol


def test_spmv_pair_matches_interpolate_spread(T):
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    op = T.make_direct_backend(pgeom(T, og))
    m = og.m
    grid = (RNG.standard_normal((m, m)) + 1j * RNG.standard_normal((m, m))).astype(np.complex64)
    # product layout is node = iy*m + ix: pass the transpose of the reference grid[ix][iy]
    s_gpu = op.spmv_w(cuda(grid.T.copy(), True)).cpu().numpy().ravel()
    assert rel(s_gpu, O.interpolate(og, grid)) < OP_TOL
    s = (RNG.standard_normal(og.P) + 1j * RNG.standard_normal(og.P)).astype(np.complex64)
    g_gpu = op.spmv_wt(cuda(s, True)).cpu().numpy()[0]
    assert rel(g_gpu.T, O.spread(og, s)) < OP_TOL


def test_batch_and_host_pointers(T):
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    op = T.make_direct_backend(pgeom(T, og), max_batch=3)
    n = og.n
    u = (RNG.standard_normal((3, n, n)) + 1j * RNG.standard_normal((3, n, n))).astype(np.complex64)
    batched = op.apply_normal(cuda(u, True)).cpu().numpy()
    for b in range(3):
        single = op.apply_normal(cuda(u[b], True)).cpu().numpy()
        assert rel(batched[b], single[0] if single.ndim == 3 else single) < 1e-6
    host = op.apply_normal(u)  # numpy in -> staged through the C ABI -> numpy out
    assert isinstance(host, np.ndarray)
    assert rel(host, batched) < 1e-6


GOLD = cases()


@pytest.fixture(params=GOLD, ids=[os.path.basename(c) for c in GOLD])
def gold(request):
    return load(request.param)


def gold_geom(T, d):
    msp = int(d["m_sp"])
    return T.Geometry(n=int(d["n"]), n_angles=int(d["n_angles"]), win_lo=-msp, win_hi=msp, tau=float(d["tau"]))


@pytest.mark.parametrize("prec", PRECS)
def test_golden_operator(T, gold, prec):
    """CUDA path vs outputs of the reference itself (tests/golden, built from /root/reference)."""
    f64 = prec == "f64"
    tol = OP_TOL_F64 if f64 else OP_TOL
    op = T.make_direct_backend(gold_geom(T, gold), precision=prec)
    assert rel(op.forward(cuda(gold["u"], True, f64)).cpu().numpy().ravel(), gold["type2_u"]) < tol
    assert rel(op.adjoint(cuda(gold["s"], True, f64)).cpu().numpy().ravel(), gold["type1_s"].ravel()) < tol
    assert rel(op.apply_normal(cuda(gold["u"], True, f64)).cpu().numpy().ravel(), gold["normal_u"].ravel()) < tol
    assert rel(op.apply_normal_real(cuda(gold["ur"], False, f64)).cpu().numpy().ravel(),
               gold["normal_real_ur"].ravel()) < tol


def test_golden_surrogate(T, gold):
    for r in (1, 2):
        op = T.make_surrogate_backend(gold_geom(T, gold), radius_r=r)
        assert rel(op.stencil(), gold[f"stencil_r{r}"]) < OP_TOL
        out = op.apply_normal_real(cuda(gold["ur"])).cpu().numpy().ravel()
        assert rel(out, gold[f"surrogate_ur_r{r}"].ravel()) < OP_TOL


def test_golden_cg(T, gold):
    op = T.make_direct_backend(gold_geom(T, gold), precision="f64")
    x, st = op.cg(cuda(gold["cg_rhs"], False, True), alpha=10.0, lambda_=1.0, steps=5)
    assert rel(x.cpu().numpy().ravel(), gold["cg_x"].ravel()) < 1e-8
    assert abs(st[0].min_ritz - float(gold["cg_min_ritz"])) < 1e-4 * abs(float(gold["cg_min_ritz"]))
    assert st[0].steps_run == 5


def test_golden_split_bregman(T, gold):
    g = gold_geom(T, gold)
    op = T.make_direct_backend(g, precision="f64")
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=5, cg_steps_per_update=5, update_tol_rel=0.0)
    mu, tr = op.split_bregman(cuda(gold["data"], True, True), cfg)
    assert rel(mu.cpu().numpy().ravel(), gold["sb_direct_mu"].ravel()) < REC_TOL
    assert rel(tr[0].update_l1, gold["sb_direct_upd"]) < REC_TOL
    assert abs(tr[0].imag_leakage - float(gold["sb_direct_leak"])) < 1e-3 * max(float(gold["sb_direct_leak"]), 1e-6) + 1e-6
    sop = T.make_surrogate_backend(g, radius_r=1)
    cfg = T.SolverConfig(alpha=1.0, lambda_=1.0, max_bregman_iters=5, cg_steps_per_update=5, update_tol_rel=0.0)
    mu, tr = sop.split_bregman(cuda(gold["data"], True), cfg)
    assert abs(tr[0].stabilization_shift - float(gold["sb_sur_sigma"])) <= 1e-3 * abs(float(gold["sb_sur_sigma"])) + 1e-9
    assert rel(mu.cpu().numpy().ravel(), gold["sb_sur_mu"].ravel()) < REC_TOL


def test_golden_tikhonov(T, gold):
    op = T.make_direct_backend(gold_geom(T, gold), precision="f64")
    mu = op.tikhonov(cuda(gold["data"], True, True), alpha=1.0, steps=20)
    assert rel(mu.cpu().numpy().ravel(), gold["tikhonov_mu"].ravel()) < REC_TOL


def test_sb_extension_geometry_and_batch(T):
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    n = og.n
    fs = []
    for seed in (1, 2):
        ph = O.random_ellipses(n, 10, seed)
        f, _ = O.synthesize(og, ph, 0.01, seed)
        fs.append(f.astype(np.complex64))
    op = T.make_direct_backend(pgeom(T, og), max_batch=2, precision="f64")
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=6, cg_steps_per_update=4, update_tol_rel=0.0)
    mu, tr = op.split_bregman(cuda(np.stack(fs), True, True), cfg)
    for b in range(2):
        ref, upd, _ = O.split_bregman(og, fs[b], backend=0, alpha=10.0, lam=1.0, max_iters=6, cg_steps=4)
        assert rel(mu[b].cpu().numpy(), ref) < REC_TOL
        assert tr[b].iterations == 6


def test_sb_tolerance_stop(T):
    og = O.Geometry(**GEOMS["ref_msp6"])
    ph = O.shepp_logan(og.n)
    f, _ = O.synthesize(og, ph, 0.0, 0)
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    cfg = T.SolverConfig(alpha=1.0, lambda_=1.0, max_bregman_iters=40, cg_steps_per_update=5, update_tol_rel=0.05)
    mu, tr = op.split_bregman(cuda(f, True, True), cfg)
    ref, upd, otr = O.split_bregman(og, f, backend=0, alpha=1.0, lam=1.0, max_iters=40,
                                    cg_steps=5, update_tol_rel=0.05)
    assert tr[0].stopping_reason == "tolerance" and otr.stopped_on_tolerance == 1
    assert tr[0].iterations == otr.iterations
    assert rel(mu.cpu().numpy(), ref) < REC_TOL


def test_surrogate_sb_batch_vs_oracle(T):
    og = O.Geometry(**GEOMS["n128"])
    n = og.n
    fs = []
    for seed in (3, 4, 5):
        ph = O.random_ellipses(n, 10, seed)
        f, _ = O.synthesize(og, ph, 0.01, seed)
        fs.append(f.astype(np.complex64))
    op = T.make_surrogate_backend(pgeom(T, og), radius_r=1, max_batch=3)
    cfg = T.SolverConfig(alpha=1.0, lambda_=1.0, max_bregman_iters=8, cg_steps_per_update=5, update_tol_rel=0.0)
    mu, tr = op.split_bregman(cuda(np.stack(fs), True), cfg)
    sigma = O.surrogate_sigma(og, 1, 1.0, 1.0)
    assert abs(tr[0].stabilization_shift - sigma) <= 1e-3 * sigma
    for b in range(3):
        ref, _, _ = O.split_bregman(og, fs[b], backend=2, r=1, alpha=1.0, lam=1.0, max_iters=8, cg_steps=5,
                                    sigma=tr[0].stabilization_shift)
        assert rel(mu[b].cpu().numpy(), ref) < REC_TOL


def test_chambolle_pock_vs_oracle(T):
    og = O.Geometry(**GEOMS["R4_gl_tau"])
    ph = O.random_ellipses(og.n, 6, 11)
    f, _ = O.synthesize(og, ph, 0.01, 11)
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    kw = dict(alpha=1e-2, lambda_=1e-2, tau_cp=0.35, sigma_cp=0.35, theta=1.0, iters=4, cg_steps=6)
    mu = op.chambolle_pock(cuda(f, True, True), **kw)
    ref = O.chambolle_pock(og, f, alpha=1e-2, lam=1e-2, tau_cp=0.35, sigma_cp=0.35, theta=1.0, iters=4, cg_steps=6)
    assert rel(mu.cpu().numpy(), ref) < REC_TOL


def test_angle_shards_sum_to_full(T):
    """Row sharding by angle blocks: partial normal ops of the blocks sum to the full one."""
    og = O.Geometry(**GEOMS["width6_odd_nb"])
    g = pgeom(T, og)
    full = T.make_direct_backend(g)
    A = og.n_angles
    parts = [T.make_direct_backend(g, angle_block=(0, A // 3)), T.make_direct_backend(g, angle_block=(A // 3, A))]
    for p in parts:
        p.set_allreduce(lambda buf, count, stream: None)  # single process: no peers to sum with
    u = RNG.standard_normal((og.n, og.n)).astype(np.float32)
    tot = sum(p.apply_normal_real(cuda(u)).cpu().numpy() for p in parts)
    assert rel(tot, full.apply_normal_real(cuda(u)).cpu().numpy()) < 1e-6


@pytest.mark.parametrize("prec", PRECS)
def test_grad_shrink_ops(T, prec):
    f64 = prec == "f64"
    n = 33
    u = RNG.standard_normal((n, n))
    if not f64:
        u = u.astype(np.float32)
    gx, gy = T.grad(cuda(u, False, f64))
    ogx, ogy = O.grad(u.astype(np.float64))
    assert np.allclose(gx.cpu().numpy(), ogx, atol=1e-6) and np.allclose(gy.cpu().numpy(), ogy, atol=1e-6)
    adj = T.grad_adjoint(gx, gy).cpu().numpy()
    assert np.allclose(adj, O.grad_adjoint(ogx, ogy), atol=1e-5)
    sh = T.shrink(cuda(u, False, f64), 0.5).cpu().numpy()
    assert np.allclose(sh, O.shrink(u.astype(np.float64), 0.5), atol=1e-6)


def test_config_errors_are_raised(T):
    with pytest.raises(T.ConfigError):
        T.make_direct_backend(T.Geometry(n=30, n_angles=4))  # m = 60 not a power of two
    with pytest.raises(T.ConfigError):
        T.make_surrogate_backend(T.Geometry(n=32, n_angles=4), radius_r=7)
    op = T.make_direct_backend(T.Geometry(n=32, n_angles=8))
    with pytest.raises(T.ConfigError):
        op.apply_normal(cuda(np.zeros((31, 31)), True))


def test_full_size_properties(T):
    """c3-sized operator (1024^2, 180 x 1449, width 6): adjointness and self-adjointness of N,
    checked without the oracle (size-independent properties)."""
    g = T.Geometry(n=1024, n_angles=180, n_b=1449, win_lo=-2, win_hi=3, tau=3 / 1024 ** 2)
    op = T.make_direct_backend(g)
    gen = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(1024, 1024, dtype=torch.complex64, device="cuda", generator=gen)
    v = torch.randn(1024, 1024, dtype=torch.complex64, device="cuda", generator=gen)
    s = torch.randn(g.P, dtype=torch.complex64, device="cuda", generator=gen)
    fu = op.forward(u)
    lhs = torch.vdot(s.to(torch.complex128), fu.reshape(-1).to(torch.complex128))
    rhs = torch.vdot(op.adjoint(s).reshape(-1).to(torch.complex128), u.reshape(-1).to(torch.complex128))
    assert abs(lhs - rhs) / abs(lhs) < 1e-5
    nu, nv = op.apply_normal(u), op.apply_normal(v)
    a = torch.vdot(v.reshape(-1).to(torch.complex128), nu.reshape(-1).to(torch.complex128))
    b = torch.vdot(nv.reshape(-1).to(torch.complex128), u.reshape(-1).to(torch.complex128))
    assert abs(a - b) / abs(a) < 1e-5
    # linearity
    w = op.apply_normal(u + 2 * v)
    assert (torch.linalg.norm(w - (nu + 2 * nv)) / torch.linalg.norm(w)).item() < 1e-5


def test_sb_recorded_trace_vs_oracle(T):
    """Recorded split Bregman (per-iteration graphs + events): same iterate as the one-graph
    solve, update_l1 per iteration, rel_l1_err against the phantom (record_reference), and
    monotone t_total_s >= t_cg_s."""
    og = O.Geometry(**GEOMS["ref_msp3"])
    ph = O.shepp_logan(og.n)
    f, _ = O.synthesize(og, ph, 0.0, 0)
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=6, cg_steps_per_update=4, update_tol_rel=0.0)
    mu0, tr0 = op.split_bregman(cuda(f, True, True), cfg)
    mu, tr = op.split_bregman_record(cuda(f, True, True), cfg, reference=cuda(ph, False, True))
    assert np.array_equal(mu.cpu().numpy(), mu0.cpu().numpy())
    t = tr[0]
    assert t.iterations == 6 and np.allclose(t.update_l1, tr0[0].update_l1, rtol=0, atol=0)
    ref_mu, ref_upd, _ = O.split_bregman(og, f, backend=0, alpha=10.0, lam=1.0, max_iters=6, cg_steps=4)
    assert rel(t.update_l1, ref_upd) < REC_TOL
    assert abs(t.rel_l1_err[-1] - O.rel_l1(mu[0].cpu().numpy(), ph)) < 1e-12
    assert np.all(np.diff(t.t_total_s) > 0) and np.all(t.t_cg_s <= t.t_total_s) and np.all(np.diff(t.t_cg_s) > 0)
    # tolerance stop: logs stop at the stopping iteration
    cfg.update_tol_rel = 0.5
    cfg.max_bregman_iters = 40
    _, tr = op.split_bregman_record(cuda(f, True, True), cfg, reference=cuda(ph, False, True))
    assert tr[0].stopping_reason == "tolerance" and len(tr[0].rel_l1_err) == tr[0].iterations < 40
    # a longer recorded solve after shorter ones (the update graph is reused across solves with
    # different lengths, and the reference is always copied into op scratch): its per-iteration
    # logs equal those of a fresh op, and a different reference buffer is honoured
    cfg.update_tol_rel = 0.0
    cfg.max_bregman_iters = 12
    ref2 = cuda(0.5 * ph, False, True)
    mu_a, tr_a = op.split_bregman_record(cuda(f, True, True), cfg, reference=ref2)
    fresh = T.make_direct_backend(pgeom(T, og), precision="f64")
    mu_b, tr_b = fresh.split_bregman_record(cuda(f, True, True), cfg, reference=cuda(0.5 * ph, False, True))
    assert np.array_equal(mu_a.cpu().numpy(), mu_b.cpu().numpy())
    assert np.array_equal(tr_a[0].rel_l1_err, tr_b[0].rel_l1_err) and len(tr_a[0].rel_l1_err) == 12
    assert np.array_equal(tr_a[0].update_l1, tr_b[0].update_l1)
    assert abs(tr_a[0].rel_l1_err[-1] - O.rel_l1(mu_a[0].cpu().numpy(), 0.5 * ph)) < 1e-12


@pytest.mark.parametrize("backend", ["direct", "surrogate"])
def test_sb_data_feedback_vs_oracle(T, backend):
    """SolverConfig.data_feedback (solver.cpp:176-187, 283-286) on the GPU vs the oracle (pinned to
    the reference in tests/test_oracle_pin.py), in both the one-graph and the recorded driver."""
    og = O.Geometry(**GEOMS["ref_msp3"])
    ph = O.shepp_logan(og.n)
    f, _ = O.synthesize(og, ph, 0.0, 0)
    alpha = 10.0 if backend == "direct" else 1.0
    op = (T.make_direct_backend(pgeom(T, og), precision="f64") if backend == "direct"
          else T.make_surrogate_backend(pgeom(T, og), radius_r=1, precision="f64"))
    cfg = T.SolverConfig(alpha=alpha, lambda_=1.0, max_bregman_iters=4, cg_steps_per_update=4, update_tol_rel=0.0,
                         data_feedback=True)
    mu, tr = op.split_bregman(cuda(f, True, True), cfg)
    mref, uref, rtr = O.split_bregman(og, f, backend=0 if backend == "direct" else 2, alpha=alpha, lam=1.0,
                                      max_iters=4, cg_steps=4, feedback=True)
    assert rel(mu[0].cpu().numpy(), mref) < REC_TOL
    assert rel(tr[0].update_l1, uref) < REC_TOL
    if backend == "surrogate":
        assert abs(tr[0].stabilization_shift - rtr.sigma) <= 1e-3 * abs(rtr.sigma)
    mu2, tr2 = op.split_bregman_record(cuda(f, True, True), cfg)
    assert np.array_equal(mu2.cpu().numpy(), mu.cpu().numpy())


@pytest.mark.parametrize("tol", [0.0, 3e-2, 1e-3])
def test_cg_exits_vs_oracle(T, tol):
    """cg_solve's exits (solver.cpp:70,75,86-88) through the Chronopoulos-Gear form: the relative
    tolerance stop, rs == 0 (zero right-hand side) and the fixed step count, per slice of a batch;
    steps_run / final_rs / min_ritz / x against the oracle's standard CG."""
    og = O.Geometry(**GEOMS["ref_msp3"])
    n = og.n
    op = T.make_direct_backend(pgeom(T, og), precision="f64")
    # alpha N + lambda K'K + I: well conditioned, so the tolerances stop it at 5 / 10 steps
    sysd = O.system(0, alpha=1e-3, lam=0.1, shift=1.0)
    rhs = np.stack([RNG.standard_normal((n, n)), np.zeros((n, n)), RNG.standard_normal((n, n))])
    x, st = op.cg(cuda(rhs, False, True), alpha=1e-3, lambda_=0.1, shift=1.0, steps=12, rel_tol=tol)
    x = x.cpu().numpy()
    for b in range(3):
        xr, sr = O.cg(og, sysd, rhs[b], steps=12, rel_tol=tol)
        assert st[b].steps_run == sr.steps_run
        if b == 1:
            assert sr.steps_run == 0 and not np.any(x[b])
            continue
        assert rel(x[b].ravel(), np.asarray(xr).ravel()) < 1e-8
        assert abs(st[b].final_rs - sr.final_rs) <= 1e-6 * sr.final_rs
        assert abs(st[b].min_ritz - sr.min_ritz) <= 1e-8 * abs(sr.min_ritz)
    if tol > 0:
        assert 0 < st[0].steps_run < 12  # the tolerance stop is exercised

