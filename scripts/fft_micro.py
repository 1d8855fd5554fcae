"""Micro-benchmark of the in-CTA FFT rows (tomo_fft_rows) vs a device copy: GB/s for rows x m."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1705_07497_b200 as T

def bench(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps

for dt in (torch.complex64, torch.complex128):
    for m, rows in ((1024, 1024), (1024, 16384), (2048, 2048), (2048, 8192), (8192, 2048)):
        x = torch.randn(rows, m, dtype=dt, device='cuda')
        y = torch.empty_like(x)
        nbytes = 2 * x.numel() * x.element_size()
        ms = bench(lambda: T.tomo.fft_rows(x))
        ms_c = bench(lambda: y.copy_(x))
        print(f'{str(dt):16s} m={m:5d} rows={rows:6d}  fft {ms*1e3:8.1f} us {nbytes/ms/1e6:7.0f} GB/s   copy {ms_c*1e3:7.1f} us {nbytes/ms_c/1e6:7.0f} GB/s', flush=True)
