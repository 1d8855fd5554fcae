"""Diagnostic: conditioning of the c5 Chambolle-Pock prox system (I + tau*alpha*N) vs GPU/oracle
agreement. For each alpha: lambda_max estimate of tau*alpha*N, GPU CG (both CG forms) vs the
oracle's CG after k steps, and one CP iteration vs the oracle."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1705_07497_b200 as T
from oracle import oracle as O

c = bench.CONFIGS["c5"]
g = bench.make_geom(T, c)
og = O.Geometry(n=g.n, n_angles=g.n_angles, n_b=g.n_b, oversample=g.oversample, win_lo=g.win_lo, win_hi=g.win_hi, tau=g.tau)
ph = O.random_ellipses(g.n, 10, 5000)
f, _ = O.synthesize(og, ph, 0.01, 5000)
op = T.make_direct_backend(g, precision="f64")
fd = torch.from_numpy(f).cuda()
bp1 = O.backproject(og, 0, 1.0, f)
for alpha in [float(a) for a in sys.argv[1:]]:
    ta = c["tau_cp"] * alpha
    rhs = c["tau_cp"] * alpha * bp1
    sysd = O.system(backend=0, alpha=ta, lam=0.0, shift=0.0, identity_k=True)
    for k in (1, 5, 10, 15):
        x, st = op.cg(torch.from_numpy(rhs).cuda(), alpha=ta, lambda_=0.0, shift=1.0, steps=k)
        xo, sto = O.cg(og, sysd, rhs, steps=k)
        print(f"alpha {alpha:g} k {k} gpu-vs-oracle CG rel {np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo):.3e} "
              f"ritz {st[0].min_ritz:.6g} / {sto.min_ritz:.6g}", flush=True)
    mu = op.chambolle_pock(fd, alpha=alpha, lambda_=c["lam"] * alpha / 1e-3, tau_cp=c["tau_cp"], sigma_cp=c["sigma_cp"],
                           theta=c["theta"], iters=1, cg_steps=c["cg"]).cpu().numpy()
    ref = O.chambolle_pock(og, f, alpha=alpha, lam=c["lam"] * alpha / 1e-3, tau_cp=c["tau_cp"], sigma_cp=c["sigma_cp"],
                           theta=c["theta"], iters=1, cg_steps=c["cg"])
    mu2 = op.chambolle_pock(fd, alpha=alpha, lambda_=c["lam"] * alpha / 1e-3, tau_cp=c["tau_cp"], sigma_cp=c["sigma_cp"],
                            theta=c["theta"], iters=4, cg_steps=c["cg"]).cpu().numpy()
    print(f"alpha {alpha:g} CP 1x15 rel {np.linalg.norm(mu - ref) / np.linalg.norm(ref):.3e}; "
          f"CP 4x15 rel-L1 vs phantom {np.abs(mu2 - ph).sum() / np.abs(ph).sum():.4f}", flush=True)
