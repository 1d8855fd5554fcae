"""Config-scale reconstruction parity: GPU (fp32) vs the fp64 oracle on BASELINE configs."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1705_07497_b200 as T
from oracle import oracle as O


def rel(a, b):
    a = np.asarray(a, np.float64).ravel(); b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def geoms(n, A, nb):
    og = O.Geometry(n=n, n_angles=A, n_b=nb, win_lo=-2, win_hi=3, tau=3.0 / n ** 2)
    g = T.Geometry(n=n, n_angles=A, n_b=nb, win_lo=-2, win_hi=3, tau=3.0 / n ** 2)
    return og, g


which = sys.argv[1:] or ['c1', 'c2', 'c4']
if 'c1' in which:
    og, g = geoms(256, 60, 367)
    ph = O.random_ellipses(256, 10, 1); f, _ = O.synthesize(og, ph, 0.01, 1); f = f.astype(np.complex64)
    op = T.make_direct_backend(g, precision='f64')
    t = time.time(); ref = O.tikhonov_identity(og, f, alpha=1.0, steps=20); tc = time.time() - t
    mu = op.tikhonov(torch.from_numpy(f.astype(np.complex128)).cuda(), alpha=1.0, steps=20).cpu().numpy()
    print('c1 tikhonov 20 CG: rel', rel(mu, ref), 'oracle s', tc, flush=True)
if 'c4' in which:
    og, g = geoms(512, 120, 725)
    ph = O.random_ellipses(512, 10, 4); f, _ = O.synthesize(og, ph, 0.01, 4); f = f.astype(np.complex64)
    op = T.make_surrogate_backend(g, radius_r=1)
    cfg = T.SolverConfig(alpha=1.0, lambda_=1.0, max_bregman_iters=30, cg_steps_per_update=5, update_tol_rel=0.0)
    mu, tr = op.split_bregman(torch.from_numpy(f).cuda(), cfg)
    t = time.time()
    ref, upd, otr = O.split_bregman(og, f, backend=2, r=1, alpha=1.0, lam=1.0, max_iters=30, cg_steps=5,
                                    sigma=tr[0].stabilization_shift)
    print('c4 surrogate SB 30x5: rel', rel(mu.cpu().numpy(), ref), 'sigma gpu', tr[0].stabilization_shift,
          'oracle s', time.time() - t, 'rel-L1 vs phantom gpu/oracle', O.rel_l1(mu.cpu().numpy(), ph), O.rel_l1(ref, ph), flush=True)
    s_or = O.surrogate_sigma(og, 1, 1.0, 1.0)
    print('c4 sigma oracle', s_or, flush=True)
if 'c2' in which:
    og, g = geoms(512, 90, 725)
    ph = O.random_ellipses(512, 10, 2); f, _ = O.synthesize(og, ph, 0.01, 2); f = f.astype(np.complex64)
    op = T.make_direct_backend(g, precision='f64')
    f = f.astype(np.complex128)
    for iters in (1, 5, 50):
        cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=iters, cg_steps_per_update=10, update_tol_rel=0.0)
        mu, tr = op.split_bregman(torch.from_numpy(f).cuda(), cfg)
        t = time.time()
        ref, upd, otr = O.split_bregman(og, f, backend=0, alpha=10.0, lam=1.0, max_iters=iters, cg_steps=10)
        print('c2 SB', iters, 'x10: rel', rel(mu.cpu().numpy(), ref), 'oracle s', time.time() - t,
              'rel-L1 vs phantom gpu/oracle', O.rel_l1(mu.cpu().numpy(), ph), O.rel_l1(ref, ph), flush=True)
