"""Small driver for ncu: builds a config's operator and runs a few normal-op applies (and,
for SB configs, a few CG steps) outside CUDA graphs so every kernel launch is visible."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1705_07497_b200 as T
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else 'c3'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = bench.CONFIGS[cfg]
g = bench.make_geom(T, c)
if c['kind'] == 'sb_sur':
    op = T.make_surrogate_backend(g, radius_r=c['r'], max_batch=32)
    f = torch.zeros(32, g.n, g.n, dtype=torch.float32, device='cuda')
    for _ in range(reps):
        op.profile_stages(batch=32, reps=1)
else:
    op = T.make_direct_backend(g, precision=c['prec'])
    dt = torch.complex128 if op.f64 else torch.complex64
    u = torch.randn(g.n, g.n, dtype=dt, device='cuda')
    for _ in range(reps):
        v = op.apply_normal(u)
    for _ in range(reps):
        op.profile_stages(batch=1, reps=1)
torch.cuda.synchronize()
print('ok', cfg, T.kernel_launches())
