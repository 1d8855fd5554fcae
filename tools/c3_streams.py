"""A/B: c3 applies on K streams, each graph-captured; `python tools/c3_streams.py K [shared]` uses K
op handles, or ONE shared op serving all K streams (reentrant: one workspace per stream)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1705_07497_b200 as T
from bench import CONFIGS, make_geom

c = CONFIGS["c3"]
g = make_geom(T, c)
nops = int(sys.argv[1]) if len(sys.argv) > 1 else 2
shared = len(sys.argv) > 2 and sys.argv[2] == "shared"
if shared:
    op0 = T.make_direct_backend(g, precision="f32")
    ops = [op0] * nops
else:
    ops = [T.make_direct_backend(g, precision="f32") for _ in range(nops)]
u = torch.randn(g.n, g.n, dtype=torch.complex64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(nops)]
applies, chunk = 1000, 50
per = applies // nops
graphs = []
for op, s in zip(ops, streams):
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            op.apply_normal(u)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s, capture_error_mode="relaxed"):
        for _ in range(chunk):
            op.apply_normal(u)
    graphs.append(gr)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for k in range(per // chunk):
        for gr, s in zip(graphs, streams):
            with torch.cuda.stream(s):
                gr.replay()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"streams={nops} {'one shared op' if shared else 'ops=' + str(nops)} applies/s {applies / (ms * 1e-3):.0f}")
