import torch, time
N = 8 << 20
h_in = torch.empty(N * 50, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N * 50, dtype=torch.uint8).pin_memory()
d = torch.empty(N * 50, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ["h2d", "d2h", "both"]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    for rep in range(3):
        for i in range(50):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d[i * N:(i + 1) * N].copy_(h_in[i * N:(i + 1) * N], non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_out[i * N:(i + 1) * N].copy_(d[i * N:(i + 1) * N], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(mode, "GB/s per direction", 3 * 50 * N / dt / 1e9)
