"""Apply the normal operator of a bench config to a fixed random input and save the output
(A/B correctness check of build/env variants): python tools/ab_apply.py c5 out.npy"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1705_07497_b200 as T
from bench import CONFIGS, make_geom

c = CONFIGS[sys.argv[1]]
g = make_geom(T, c)
op = T.make_direct_backend(g, precision=c["prec"])
rng = np.random.default_rng(0)
u = rng.standard_normal((g.n, g.n))
dt = torch.float64 if c["prec"] == "f64" else torch.float32
out = op.apply_normal_real(torch.from_numpy(u).to(dt).cuda()).cpu().numpy()
np.save(sys.argv[2], out[::4, ::4])  # subsample: keeps gpurun_out small
print(sys.argv[1], float(np.linalg.norm(out)))
