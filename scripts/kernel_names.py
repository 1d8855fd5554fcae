"""List the library kernels one normal-operator apply launches (torch profiler / CUPTI names)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1705_07497_b200 as T

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
g = bench.make_geom(T, c)
op = T.make_direct_backend(g, precision=c["prec"])
u = torch.randn(g.n, g.n, dtype=torch.float64 if c["prec"] == "f64" else torch.float32, device="cuda")
op.apply_normal_real(u)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    op.apply_normal_real(u)
    torch.cuda.synchronize()
for e in prof.key_averages():
    if e.device_type == torch.autograd.DeviceType.CUDA or "k_" in e.key:
        print(f"{e.key[:90]:90s} {e.device_time_total if hasattr(e, 'device_time_total') else e.cuda_time_total:.1f}")
