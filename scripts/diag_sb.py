import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1705_07497_b200 as T
from oracle import oracle as O
from tests.golden_util import load, rel
for name in ['ref_n32_msp3', 'ref_n32_msp6', 'ref_n64_msp2']:
    d = load(f'tests/golden/{name}.npz'); msp = int(d['m_sp'])
    og = O.Geometry(n=int(d['n']), n_angles=int(d['n_angles']), win_lo=-msp, win_hi=msp, tau=float(d['tau']))
    g = T.Geometry(n=og.n, n_angles=og.n_angles, win_lo=-msp, win_hi=msp, tau=og.tau)
    op = T.make_direct_backend(g)
    f = d['data'].astype(np.complex64)
    ft = torch.from_numpy(f).cuda()
    for it in (1, 2, 3, 5):
        cfg = T.SolverConfig(alpha=10.0, lambda_=1.0, max_bregman_iters=it, cg_steps_per_update=5, update_tol_rel=0.0)
        mu, tr = op.split_bregman(ft, cfg)
        ref, upd, _ = O.split_bregman(og, f, backend=0, alpha=10, lam=1, max_iters=it, cg_steps=5)
        print(name, 'iters', it, 'mu rel', rel(mu.cpu().numpy(), ref), 'upd rel', rel(tr[0].update_l1, upd))
    # CG sensitivity: cg from random x0 on the SB system, 5 and 10 steps
    rng = np.random.default_rng(0)
    b = rng.standard_normal((og.n, og.n)); x0 = rng.standard_normal((og.n, og.n))
    for steps in (1, 3, 5, 10):
        x, st = op.cg(torch.from_numpy(b.astype(np.float32)).cuda(), torch.from_numpy(x0.astype(np.float32)).cuda(), alpha=10.0, lambda_=1.0, steps=steps)
        xr, sr = O.cg(og, O.system(0, alpha=10.0, lam=1.0), b.astype(np.float32), x0.astype(np.float32), steps=steps)
        print(name, 'cg steps', steps, rel(x.cpu().numpy(), xr), st[0].min_ritz, sr.min_ritz)
    # backprojection
    bp = op.backproject(ft, alpha=10.0).cpu().numpy()
    print(name, 'bp', rel(bp, O.backproject(og, 0, 10.0, f)))
