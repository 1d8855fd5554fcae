"""Run a few split-Bregman solves of a bench config (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1705_07497_b200 as T
import bench
cfg = sys.argv[1] if len(sys.argv) > 1 else 'c2'
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = dict(bench.CONFIGS[cfg]); c['iters'] = iters
wl = bench.Workload(cfg, c, 1, 0, 0, torch)
for _ in range(2):
    wl.step()
torch.cuda.synchronize()
print('ok', T.kernel_launches())
