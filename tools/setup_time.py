"""Operator construction time (host plan + W / W^T / Gram tables + upload) per BASELINE config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_07497_b200 as T  # noqa: E402
from bench import CONFIGS, make_geom  # noqa: E402

torch.cuda.init()
for name in sys.argv[1:] or ("c2", "c3", "c5"):
    c = CONFIGS[name]
    t = time.perf_counter()
    op = T.make_direct_backend(make_geom(T, c), precision=c["prec"])
    print(name, "direct build s", round(time.perf_counter() - t, 2), flush=True)
    del op
t = time.perf_counter()
op = T.make_fused_backend(make_geom(T, CONFIGS["c2"]), precision="f64")
print("c2 fused build s", round(time.perf_counter() - t, 2), "gram nnz", op.info.gram_nnz, flush=True)
