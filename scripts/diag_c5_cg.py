"""Diagnostic: GPU CG (TOMO_AB=1 TOMO_CG=std selects the standard form) vs the oracle's CG on the
c5 prox system (I + tau*alpha*N) u = tau*alpha*Re(F_NU f), after k steps; and the oracle's own
spread under rounding-level perturbations (orc_set_perturbation)."""
import os, sys
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
alpha = c["alpha"]
ta = c["tau_cp"] * alpha
rhs = ta * O.backproject(og, 0, 1.0, f)
sysd = O.system(backend=0, alpha=ta, lam=0.0, shift=0.0, identity_k=True)
form = "std" if os.environ.get("TOMO_CG") == "std" else "chronopoulos-gear"
for k in [int(a) for a in sys.argv[1:]] or [10, 12, 13, 14, 15]:
    x, st = op.cg(torch.from_numpy(rhs).cuda(), alpha=ta, lambda_=0.0, shift=1.0, steps=k)
    xo, sto = O.cg(og, sysd, rhs, steps=k)
    O.set_perturbation(1e-16, 5)
    xp, _ = O.cg(og, sysd, rhs, steps=k)
    O.set_perturbation(0.0)
    x = x.cpu().numpy().reshape(xo.shape)
    np.save(f"gpurun_out/diag_cg_x_{form}_{k}.npy", x[::8, ::8])
    print(f"{form} k {k}: gpu-vs-oracle {np.linalg.norm(x - xo) / np.linalg.norm(xo):.3e}  oracle spread "
          f"{np.linalg.norm(xp - xo) / np.linalg.norm(xo):.3e}  rs {st[0].final_rs:.10g} / {sto.final_rs:.10g}",
          flush=True)
