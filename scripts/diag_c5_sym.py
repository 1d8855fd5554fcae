"""Diagnostic: symmetry of Re(N) at the c5 geometry and the CG iterate history of the prox
system (I + tau*alpha*N) u = tau*alpha*Re(F_NU f) (GPU, fp64)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1705_07497_b200 as T
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
c = bench.CONFIGS["c5"]
c = dict(c, n=n, A=max(8, c["A"] * n // 2048), nb=(c["nb"] - 1) * n // 2048 + 1)
g = bench.make_geom(T, c)
og = O.Geometry(n=g.n, n_angles=g.n_angles, n_b=g.n_b, oversample=g.oversample, win_lo=g.win_lo, win_hi=g.win_hi, tau=g.tau)
op = T.make_direct_backend(g, precision="f64")
rng = np.random.default_rng(1)
u = torch.from_numpy(rng.standard_normal((n, n))).cuda()
v = torch.from_numpy(rng.standard_normal((n, n))).cuda()
Nu = op.apply_normal_real(u)
Nv = op.apply_normal_real(v)
a, b = float((v * Nu).sum()), float((Nv * u).sum())
print(f"n {n}: <v,Nu> {a:.17g} <Nv,u> {b:.17g} rel asym {abs(a - b) / abs(a):.3e}; <u,Nu> {float((u * Nu).sum()):.6g}")
ph = O.random_ellipses(n, 10, 5000)
f, _ = O.synthesize(og, ph, 0.01, 5000)
alpha = 1e-3
ta = c["tau_cp"] * alpha
bp = op.backproject(torch.from_numpy(f).cuda(), alpha=1.0)[0]
rhs = ta * bp
phd = torch.from_numpy(ph).cuda()
print("rel-L2 |Re N ph - bp| / |bp| (noise level)", float((op.apply_normal_real(phd)[0] - bp).norm() / bp.norm()))
for k in range(1, 16):
    x, st = op.cg(rhs, alpha=ta, lambda_=0.0, shift=1.0, steps=k)
    x = x[0]
    r = rhs - (ta * op.apply_normal_real(x)[0] + x)
    print(f"k {k:2d} |x| {float(x.norm()):.6g} |r|/|b| {float(r.norm() / rhs.norm()):.3e} rel-L1 vs phantom "
          f"{float((x - phd).abs().sum() / phd.abs().sum()):.4f} rs {st[0].final_rs:.6g}", flush=True)
