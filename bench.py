#!/usr/bin/env python
"""bench.py — B200 throughput of the CT normal-operator hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workloads (BASELINE.json "configs"; synthetic seeded inputs):
  c2 (default, configs[1]): 512^2 random-ellipse slice, 90 angles x 725 bins, 1% noise; TV split
      Bregman alpha=10, lambda=1, 50 outer x 10 CG on the W/W^T operator, fp64 (complex128);
      one step = one slice solved per rank (independent slices: replicas, weak scaling).
  c1: 256^2, 60 x 367; 100 normal-op applies + 20 CG on (alpha N + I) u = b (fp64).
  c3: 1024^2 complex64 operator, 180 x 1449, 2048^2 grid; one step = 1000 applies (fp32).
  c4: 256 slices 512^2, 120 x 725, surrogate r=1 split Bregman 30 x 5 (fp32), slices sharded
      across ranks (strong scaling, no collective).
Every rank prints nothing but rank 0's single JSON line. `--impl reference` times the
reference's own CPU code (oracle/_ref, the reference sources built here; else the oracle
port) on a bounded sample and prints the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent

CONFIGS = {
    # the 100 independent applies are issued as calls of 20 inputs (run on the library's lanes)
    "c1": dict(n=256, A=60, nb=367, R=2, lo=-2, hi=3, kind="c1", alpha=1.0, applies=100, batch=20, cg=20, prec="f64",
               metric="normal-op applies/sec", unit="applies/s"),
    # the reference's own m_sp = 3 window ([-3, 3], 7x7, tau = 3/n^2): BASELINE c2 states no width,
    # so both arms run the same operator (same_config with the --impl reference arm)
    "c2": dict(n=512, A=90, nb=725, R=2, lo=-3, hi=3, kind="sb", alpha=10.0, lam=1.0, iters=50, cg=10, prec="f64",
               metric="split-Bregman slices/sec", unit="slices/s"),
    # 1000 applies on random-normal inputs, issued as calls of 3 independent inputs that the
    # library runs on three concurrent lanes (streams with their own grids)
    "c3": dict(n=1024, A=180, nb=1449, R=2, lo=-2, hi=3, kind="apply", applies=1000, batch=3, prec="f32",
               metric="normal-op applies/sec", unit="applies/s"),
    "c4": dict(n=512, A=120, nb=725, R=2, lo=-2, hi=3, kind="sb_sur", alpha=1.0, lam=1.0, iters=30, cg=5, r=1,
               slices=256, prec="f32", metric="split-Bregman slices/sec", unit="slices/s"),
    # 4x oversampling (m = 8192), Greengard-Lee tau (extension D7); Chambolle-Pock with a 15-step CG
    # prox; one step = 2 CP iterations; reported as normal-op applies/s (16 applies per CP iteration)
    "c5": dict(n=2048, A=360, nb=2897, R=4, lo=-2, hi=3, kind="cp", alpha=1e-3, lam=1e-2, tau_cp=0.35,
               sigma_cp=0.35, theta=1.0, iters=2, cg=15, prec="f64", metric="normal-op applies/sec", unit="applies/s"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- distributed
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def launcher_cmd(gpus: int, argv):
    """torchrun command running `bench.py argv` as `gpus` ranks on this node (127.0.0.1)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workloads
def make_geom(T, c):
    tau = 3.0 / c["n"] ** 2 if c["R"] == 2 else None
    kw = dict(n=c["n"], n_angles=c["A"], n_b=c["nb"], oversample=c["R"], win_lo=c["lo"], win_hi=c["hi"])
    if tau:
        kw["tau"] = tau
    return T.Geometry(**kw)


def synth_slices(T, op, c, seeds, torch):
    """Random-ellipse phantoms -> F_NU^* on the GPU -> + complex Gaussian noise, sigma = 1% max|f|."""
    n = c["n"]
    out = []
    for s in seeds:
        ph = T.random_ellipses(n, 10, seed=s)
        img = torch.from_numpy(ph.astype(np.complex128 if op.f64 else np.complex64)).cuda()
        f = op.forward(img)[0].cpu().numpy()
        sigma = 0.01 * np.abs(f).max()
        rng = np.random.default_rng(10_000 + s)
        f = f + sigma * (rng.standard_normal(f.shape) + 1j * rng.standard_normal(f.shape))
        out.append(f.astype(np.complex128 if op.f64 else np.complex64))
    return np.stack(out)


class Workload:
    """One bench config on one rank: step() runs the hot path with inputs resident in HBM,
    step_e2e() the same through the C ABI with pinned host buffers."""

    def __init__(self, cfg_name, c, world, rank, local, torch):
        import paper_1705_07497_b200 as T
        self.T, self.c, self.torch = T, c, torch
        self.replayed_launches = 0  # kernels launched by torch-graph replays (not seen by the C ABI counter)
        self.sharded = False  # c5 at N > 1: one slice, angle-block sharded (strong scaling)
        self.name = cfg_name
        g = make_geom(T, c)
        self.geom = g
        kind = c["kind"]
        self.units_per_step = 1
        self.h2d = self.d2h = 0
        if kind == "sb":
            # `batch` independent slices per step, solved together (slice pairs on grid.y)
            self.batch = int(c.get("batch", 1))
            self.op = T.make_direct_backend(g, precision=c["prec"], device=local, max_batch=self.batch)
            seeds = [1000 + rank * self.batch + i for i in range(self.batch)]
            self.f = torch.from_numpy(synth_slices(T, self.op, c, seeds, torch)).cuda()
            self.units_per_step = self.batch
            self.cfg = T.SolverConfig(alpha=c["alpha"], lambda_=c["lam"], max_bregman_iters=c["iters"],
                                      cg_steps_per_update=c["cg"], update_tol_rel=0.0)
            self.f_host = self.f.cpu().pin_memory()
            self.h2d = self.f.numel() * self.f.element_size()
            self.d2h = self.batch * g.n * g.n * (8 if self.op.f64 else 4)
        elif kind == "sb_sur":
            per_rank = (c["slices"] + world - 1) // world
            lo = rank * per_rank
            hi = min(c["slices"], lo + per_rank)
            self.nslices = max(0, hi - lo)
            self.batch = min(int(c.get("batch", 64)), max(1, self.nslices))
            self.op = T.make_surrogate_backend(g, radius_r=c["r"], max_batch=self.batch, device=local)
            fs = synth_slices(T, self.op, c, list(range(2000 + lo, 2000 + hi)), torch)
            self.f = torch.from_numpy(fs).cuda()
            self.cfg = T.SolverConfig(alpha=c["alpha"], lambda_=c["lam"], max_bregman_iters=c["iters"],
                                      cg_steps_per_update=c["cg"], update_tol_rel=0.0)
            self.op.split_bregman(self.f[:1], self.cfg)  # sigma (Lanczos) is per geometry: setup
            self.units_per_step = self.nslices
            self.f_host = self.f.cpu().pin_memory()
            self.h2d = self.f.numel() * self.f.element_size()
            self.d2h = self.nslices * g.n * g.n * 4
        elif kind == "apply":
            # `batch` independent random-normal inputs per call (1 = the reference's time_apply shape)
            self.batch = int(c.get("batch", 1))
            self.op = T.make_direct_backend(g, precision=c["prec"], device=local, max_batch=self.batch)
            gen = torch.Generator(device="cuda").manual_seed(7 + rank)
            self.u = torch.randn(self.batch, g.n, g.n, dtype=torch.complex64, device="cuda", generator=gen)
            self.out = torch.empty_like(self.u)
            self.units_per_step = c["applies"]
            self.calls = c["applies"] // self.batch
            self.rem = c["applies"] % self.batch  # a last, smaller call
            self.chunk = max(d for d in range(1, 51) if self.calls % d == 0)
            self.graph = None
            # end to end: host batches of up to 50 pinned slices per call; the library streams them
            # (host->device of slice i+1 and device->host of slice i-1 overlap the apply of slice i)
            self.e2e_batch = max(d for d in range(1, 51) if c["applies"] % d == 0)
            self.u_host = self.u[0].expand(self.e2e_batch, g.n, g.n).contiguous().cpu().pin_memory()
            self.h2d = self.d2h = g.n * g.n * 8 * c["applies"]
        elif kind == "cp":
            if world > 1:
                # one large slice sharded by angle blocks: every rank owns the W rows
                # of its block; each adjoint is summed across ranks by an NCCL all-reduce inside
                # the library; the CP/CG state is replicated. Same data on every N: synthesised with
                # the whole operator, then each rank keeps its block's samples.
                from paper_1705_07497_b200.distributed import angle_blocks, make_sharded_backend
                full = T.make_direct_backend(g, precision=c["prec"], device=local)
                f_all = synth_slices(T, full, c, [5000], torch)
                del full
                a0, a1 = angle_blocks(c["A"], world)[rank]
                self.op = make_sharded_backend(g, rank, world, local, precision=c["prec"])
                self.f = torch.from_numpy(np.ascontiguousarray(f_all[:, a0 * c["nb"]:a1 * c["nb"]])).cuda()
                self.sharded = True
            else:
                self.op = T.make_direct_backend(g, precision=c["prec"], device=local)
                self.f = torch.from_numpy(synth_slices(T, self.op, c, [5000 + rank], torch)).cuda()
            self.units_per_step = c["iters"] * (c["cg"] + 1)
            self.f_host = self.f.cpu().pin_memory()
            self.h2d = self.f.numel() * self.f.element_size()
            self.d2h = g.n * g.n * 8
        elif kind == "c1":
            self.batch = int(c.get("batch", 2))
            self.op = T.make_direct_backend(g, precision=c["prec"], device=local, max_batch=self.batch)
            self.f = torch.from_numpy(synth_slices(T, self.op, c, [3000 + rank], torch)).cuda()
            ph = T.random_ellipses(g.n, 10, seed=3000 + rank)
            self.u = torch.from_numpy(ph.astype(np.float64)).cuda()
            self.u2 = self.u.expand(self.batch, g.n, g.n).contiguous()
            self.out = torch.empty_like(self.u)
            self.units_per_step = c["applies"] + c["cg"] + 1
            self.f_host = self.f.cpu().pin_memory()
            # end to end: the 100 applies as one host batch (streamed through the library)
            self.u_host = self.u.expand(c["applies"], g.n, g.n).contiguous().cpu().pin_memory()
            self.h2d = self.f.numel() * 16 + self.u_host.numel() * 8
            self.d2h = g.n * g.n * 8 * (c["applies"] + 1)
        else:
            raise SystemExit(f"unknown workload kind {kind}")

    # -- device-resident step
    def step(self):
        torch = self.torch
        k = self.c["kind"]
        if k == "sb":
            self.mu, _ = self.op.split_bregman(self.f, self.cfg)
        elif k == "sb_sur":
            for i in range(0, self.nslices, self.batch):
                self.op.split_bregman(self.f[i:i + self.batch], self.cfg)
        elif k == "apply":
            if self.graph is None:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    for _ in range(3):
                        self.op.apply_normal(self.u)
                torch.cuda.current_stream().wait_stream(s)
                self.graph = torch.cuda.CUDAGraph()
                l0 = self.T.kernel_launches()
                with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
                    for _ in range(self.chunk):
                        self.out = self.op.apply_normal(self.u)
                # our kernels captured into the torch graph: every replay launches them again
                self.per_replay = self.T.kernel_launches() - l0
            for _ in range(self.calls // self.chunk):
                self.graph.replay()
            self.replayed_launches += self.per_replay * (self.calls // self.chunk)
            if self.rem:
                self.out = self.op.apply_normal(self.u[:self.rem])
        elif k == "c1":
            # the 100 applies as calls of `batch` (independent, equal) inputs on the library's lanes
            na = self.c["applies"]
            for _ in range(na // self.batch):
                self.out = self.op.apply_normal_real(self.u2)
            if na % self.batch:
                self.out = self.op.apply_normal_real(self.u2[:na % self.batch])
            self.mu = self.op.tikhonov(self.f, alpha=self.c["alpha"], steps=self.c["cg"])
        elif k == "cp":
            c = self.c
            self.mu = self.op.chambolle_pock(self.f, alpha=c["alpha"], lambda_=c["lam"], tau_cp=c["tau_cp"],
                                             sigma_cp=c["sigma_cp"], theta=c["theta"], iters=c["iters"],
                                             cg_steps=c["cg"])

    # -- end to end through the C ABI with host (pinned) buffers
    def step_e2e(self):
        torch = self.torch
        k = self.c["kind"]
        if k == "sb":
            mu, _ = self.op.split_bregman(self.f_host, self.cfg)
        elif k == "sb_sur":
            for i in range(0, self.nslices, self.batch):
                self.op.split_bregman(self.f_host[i:i + self.batch], self.cfg)
        elif k == "apply":
            for _ in range(self.c["applies"] // self.e2e_batch):
                self.op.apply_normal(self.u_host)
        elif k == "c1":
            self.op.apply_normal_real(self.u_host)
            self.op.tikhonov(self.f_host, alpha=self.c["alpha"], steps=self.c["cg"])
        elif k == "cp":
            c = self.c
            self.op.chambolle_pock(self.f_host, alpha=c["alpha"], lambda_=c["lam"], tau_cp=c["tau_cp"],
                                   sigma_cp=c["sigma_cp"], theta=c["theta"], iters=c["iters"], cg_steps=c["cg"])

    # -- kernel census + roofline of the dominant kernel (CUDA events, live)
    def roofline(self, peak_gbs):
        c = self.c
        k = c["kind"]
        # the kernels as launched: c4 batches; c1/c3 calls of `batch` inputs run on the library's
        # lanes (TOMO_LANES, default 3) as sub-batches of ceil(batch / lanes)
        lanes = min(max(int(os.environ.get("TOMO_LANES", "3") or 3), 1), 4)
        B = self.batch if k in ("sb_sur", "sb") else (-(-self.batch // lanes) if k in ("apply", "c1") else 1)
        prof = self.op.profile_stages(batch=B, reps=10, complex_io=(k == "apply"))
        if k in ("sb", "c1", "cp"):
            steps = c.get("cg", 10)
            iters = c.get("iters", 1)
            a = iters * (steps + 1)
            counts = {"t2_rows": a, "t2_cols": a, "w_spmv": a, "wt_spread": a, "t1_cols": a, "wt_t1": a, "t1_rows": a,
                      # Chronopoulos-Gear CG (default): one update kernel per CG call, the others
                      # are fused into the next step's first FFT pass (TOMO_CG=std: one per step)
                      "cg_update": iters * steps if (os.environ.get("TOMO_AB") == "1" and os.environ.get("TOMO_CG") == "std") else iters,
                      "sb_post": iters}
        elif k == "apply":
            counts = {"t2_rows": 1, "t2_cols": 1, "w_spmv": 1, "wt_spread": 1, "t1_cols": 1, "wt_t1": 1, "t1_rows": 1}
        else:  # surrogate
            counts = {"stencil": c["iters"] * (c["cg"] + 1), "cg_update": c["iters"] * c["cg"], "sb_post": c["iters"]}
        share = {s: counts.get(s, 0) * prof[s][0] for s in prof}
        top = max(share, key=share.get)
        ms, by_run = prof[top]
        # algorithmic bytes of the dominant kernel: for the two SpMVs SURVEY §8(d)'s "SpMV metric"
        # (the reference algorithm's stage: all nnz entries, T touched nodes, the whole grid), which
        # the kernels as run undercut on the real subspace (half grid, mirror pairs: `as_run`); for
        # the other stages §8(d) has no per-stage figure and the bytes are those of the kernel as run
        by = spmv_bytes(c, self.op.info, top, B) or by_run
        achieved = by / (ms * 1e-3) / 1e9
        out = {"bound": "hbm", "kernel": top, "achieved": round(achieved, 1), "peak": peak_gbs,
               "unit": "GB/s", "frac": round(achieved / peak_gbs, 4), "traffic": None,
               "algorithmic_bytes_per_launch": int(by), "ms_per_launch": round(ms, 5),
               "bytes_formula": ("SURVEY 8(d) SpMV metric: W (4+r)nnz + cT + B cP; W^T (4+r)nnz + 8(T+1) + B(cP + cG)"
                                 if by != by_run else "kernel as run (tomo_profile_stages)"),
               "as_run": {"bytes": int(by_run), "achieved": round(by_run / (ms * 1e-3) / 1e9, 1),
                          "frac": round(by_run / (ms * 1e-3) / 1e9 / peak_gbs, 4)},
               "stage_ms": {s: round(v[0], 5) for s, v in prof.items()},
               "stage_share_of_step": {s: round(v / max(sum(share.values()), 1e-12), 4) for s, v in share.items()}}
        if k != "sb_sur":
            # the whole normal-operator apply against SURVEY §8(d)'s bytes_apply, over the sum of
            # its six stage times (live, per launch of B slices)
            stages = ("t2_rows", "t2_cols", "w_spmv", "wt_spread", "t1_cols", "t1_rows")
            t_apply = sum(prof[s][0] for s in stages if s in prof)
            ab = apply_bytes(c, self.op.info.wt_rows, complex_io=(k == "apply"), B=B)
            # the bytes the six kernels as run must move (the real-image solvers take the
            # Hermitian half grid, so they move less than SURVEY's formula)
            mb = sum(prof[s][1] for s in stages if s in prof)
            out["apply"] = {"bytes": int(ab), "ms": round(t_apply, 5), "slices_per_launch": B,
                            "achieved": round(ab / (t_apply * 1e-3) / 1e9, 1),
                            "frac": round(ab / (t_apply * 1e-3) / 1e9 / peak_gbs, 4),
                            "formula": "SURVEY 8(d): 2(4+r)nnz + 8T + B(in + out + 3cG + cT + 2cP)",
                            "moved_bytes": int(mb),
                            "moved_frac": round(mb / (t_apply * 1e-3) / 1e9 / peak_gbs, 4)}
        return top, out


def spmv_bytes(c, info, stage, B=1):
    """SURVEY.md §8(d) "SpMV metric" bytes of one W / W^T launch over B slices (None for other
    stages): every entry of the (local) matrix once per launch, the vectors once per slice."""
    if stage not in ("w_spmv", "wt_spread"):
        return None
    r = 8 if c["prec"] == "f64" else 4
    cb = 2 * r
    nnz, P, T = int(info.nnz), int(info.P), int(info.wt_rows)
    G = (c["R"] * c["n"]) ** 2
    if stage == "w_spmv":
        return (4 + r) * nnz + B * (cb * T + cb * P)
    return (4 + r) * nnz + 8 * (T + 1) + B * (cb * P + cb * G)


def apply_bytes(c, T, complex_io, B=1):
    """SURVEY.md §8(d) algorithmic bytes of one normal-operator apply: input + output images,
    pad/iFFT write + FFT read + W^T grid write (3 c G), W and W^T entry streams (2 (4 + r) nnz),
    W's gather of the T touched nodes (c T) + W^T's row pointers and ids (8 T), and the slice
    write + read (2 c P). r = real bytes, c = 2 r."""
    r = 8 if c["prec"] == "f64" else 4
    cb = 2 * r
    n2 = c["n"] ** 2
    G = (c["R"] * c["n"]) ** 2
    P = c["A"] * c["nb"]
    w = c["hi"] - c["lo"] + 1
    nnz = P * w * w
    io = 2 * n2 * (cb if complex_io else r)
    # matrix streams once per launch, vectors once per slice (B slices per launch)
    return 2 * (4 + r) * nnz + 8 * T + B * (io + 3 * cb * G + cb * T + 2 * cb * P)


def flush_l2(torch, buf):
    buf.add_(1)  # writes 256 MiB > 126 MB L2


# ----------------------------------------------------------------------------- CPU baseline
# The reference's own CPU code (oracle/_ref: the unmodified reference sources built here with its
# -O3 -march=native, proj/CMakeLists.txt:10), or the oracle port where the reference has no such
# path (c4: its surrogate weights assume n_b = n, normal_ops.cpp:208-219; c5: m = 2n is hard-coded,
# nufft.cpp:40). The reference is single-threaded, so "all host cores" = one process per core,
# each running its own independent slice / apply, concurrently; units/s = sum over workers.
SB_SAMPLE_ITERS = 5  # outer split-Bregman iterations timed per worker sample


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return model, cores


def _og(c, O):
    tau = 3.0 / c["n"] ** 2 if c["R"] == 2 else np.pi * max(c["hi"], -c["lo"]) / (c["n"] ** 2 * c["R"] * (c["R"] - 0.5))
    return O.Geometry(n=c["n"], n_angles=c["A"], n_b=c["nb"], oversample=c["R"], win_lo=c["lo"], win_hi=c["hi"],
                      tau=tau)


def ref_kind(c):
    """'reference' when the reference's own code runs this workload (symmetric window, R = 2,
    and for the surrogate n_b = n), else 'port'."""
    from oracle import refbind
    if not refbind.available() or c["R"] != 2 or c["lo"] != -c["hi"]:
        return "port"
    if c["kind"] == "sb_sur" and c["nb"] != c["n"]:
        return "port"
    if c["kind"] == "cp":
        return "port"
    return "reference"


_WORKER_STATE = {}


def _cpu_worker(job):
    """One bounded sample in a spawned process: returns (units, seconds_per_unit_extrapolated,
    wall seconds of the sample)."""
    c, kind, seed, threads = job
    os.environ["ORC_THREADS"] = str(threads)  # read once when the oracle library loads
    from oracle import oracle as O
    from oracle import refbind
    key = (json.dumps(c, sort_keys=True), kind)
    st = _WORKER_STATE.get(key)
    og = _og(c, O)
    if st is None:  # operator construction is outside every timed region
        st = {}
        if kind == "reference" and c["kind"] in ("sb", "sb_sur", "apply", "c1"):
            backend = 2 if c["kind"] == "sb_sur" else 0
            st["rb"] = refbind.RefBackend(c["n"], c["A"], c["hi"], og.tau, n_b=c["nb"], backend=backend,
                                          r=c.get("r", 1))
        _WORKER_STATE.clear()
        _WORKER_STATE[key] = st
    t_wall = time.perf_counter()
    if c["kind"] in ("sb", "sb_sur"):
        ph = O.random_ellipses(c["n"], 10, seed)
        f, _ = O.synthesize(og, ph, 0.01, seed)
        k = SB_SAMPLE_ITERS
        if kind == "reference":
            _, t_call, t_loop = st["rb"].split_bregman(f, c["alpha"], c["lam"], k, c["cg"])
        else:
            t0 = time.perf_counter()
            O.split_bregman(og, f, backend=2 if c["kind"] == "sb_sur" else 0, r=c.get("r", 1), alpha=c["alpha"],
                            lam=c["lam"], max_iters=1, cg_steps=c["cg"])
            t1 = time.perf_counter()
            O.split_bregman(og, f, backend=2 if c["kind"] == "sb_sur" else 0, r=c.get("r", 1), alpha=c["alpha"],
                            lam=c["lam"], max_iters=1 + k, cg_steps=c["cg"])
            t2 = time.perf_counter()
            t_loop = (t2 - t1) - (t1 - t0)  # k outer iterations, setup cancelled
            t_call = (t2 - t1)
        # slice = setup (make_subproblem, leak probe, back-projection) + iters x per-outer
        t_unit = (t_call - t_loop) + c["iters"] * t_loop / k
        return 1, t_unit, time.perf_counter() - t_wall
    if c["kind"] in ("apply", "c1"):
        rng = np.random.default_rng(seed)
        u = rng.standard_normal((c["n"], c["n"])) + 1j * rng.standard_normal((c["n"], c["n"]))
        if kind == "reference":
            med, _ = st["rb"].time_apply(u, reps=5)  # time_apply: 1 warm-up + median of 5
        else:
            O.apply_normal(og, u)
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                O.apply_normal(og, u)
                ts.append(time.perf_counter() - t0)
            med = statistics.median(ts)
        return 1, med, time.perf_counter() - t_wall
    if c["kind"] == "cp":
        # one real apply (the CP/CG unit of the metric) with the port's FFT rows on all threads
        u = np.random.default_rng(seed).standard_normal((c["n"], c["n"]))
        t0 = time.perf_counter()
        O.apply_normal_real(og, u)
        return 1, time.perf_counter() - t0, time.perf_counter() - t_wall
    raise SystemExit("no cpu sample for " + c["kind"])


class CpuBaseline:
    """The reference's CPU path on this box's host cores, one worker process per core (a single
    worker with threaded FFT rows for c5's one large slice)."""

    def __init__(self, c):
        self.c = c
        self.kind = ref_kind(c)
        self.model, ncores = host_cpu()
        big = c["kind"] == "cp"
        self.workers = 1 if big else ncores
        self.threads = ncores if big else 1
        self.cores = self.workers * self.threads
        import concurrent.futures as cf
        import multiprocessing as mp
        self.pool = cf.ProcessPoolExecutor(max_workers=self.workers, mp_context=mp.get_context("spawn"))
        self.seed = 0

    def step(self):
        """One concurrent sample on every worker: (metric units/s over all workers, wall s)."""
        t0 = time.perf_counter()
        jobs = [(self.c, self.kind, 1 + self.seed + w, self.threads) for w in range(self.workers)]
        self.seed += self.workers
        res = list(self.pool.map(_cpu_worker, jobs))
        wall = time.perf_counter() - t0
        return sum(u / t for u, t, _ in res), wall, res

    def close(self):
        self.pool.shutdown()

    def describe(self):
        c = self.c
        what = {
            "sb": f"split_bregman_tv on independent {c['n']}^2 slices ({c['A']}x{c['nb']}, window [{c['lo']},{c['hi']}]): "
                  f"{SB_SAMPLE_ITERS} outer x {c.get('cg')} CG timed per worker sample (the trace's loop time); "
                  f"slice = (call - loop) + {c.get('iters')} x loop/{SB_SAMPLE_ITERS}",
            "sb_sur": f"surrogate r={c.get('r')} split Bregman on independent {c['n']}^2 slices: {SB_SAMPLE_ITERS} outer x "
                      f"{c.get('cg')} CG per worker sample; slice = setup + {c.get('iters')} x per-outer",
            "apply": f"time_apply (1 warm-up + median of 5 complex apply_normal, backend prebuilt) at {c['n']}^2",
            "c1": f"time_apply (1 warm-up + median of 5 complex apply_normal, backend prebuilt) at {c['n']}^2; "
                  f"rate = applies/s",
            "cp": f"one real apply_normal at {c['n']}^2, R={c['R']} (m={c['R'] * c['n']}), FFT rows on all threads",
        }[c["kind"]]
        return (f"{what}; {self.workers} worker process(es) x {self.threads} thread(s) concurrently on "
                f"{self.model}; kind={self.kind}")


# ----------------------------------------------------------------------------- line helpers
DATA = "synthetic (seeded random ellipses, 1% complex Gaussian noise; c3 random normal)"


def scaling_of(c, world):
    return "strong" if (c["kind"] == "sb_sur" or (c["kind"] == "cp" and world > 1)) else "weak"


def config_dict(name, c, world):
    """The workload as both arms (ours and --impl reference) report it."""
    w = c["hi"] - c["lo"] + 1
    P = c["A"] * c["nb"]
    par = {"sb_sur": "slice-sharded", "cp": "angle-sharded" if world > 1 else "replicas"}.get(c["kind"], "replicas")
    return {"workload": name, "n": c["n"], "angles": c["A"], "n_b": c["nb"], "oversample": c["R"],
            "window": [c["lo"], c["hi"]], "m": c["R"] * c["n"], "P": P, "nnz_W": P * w * w, "precision": c["prec"],
            **{k: c[k] for k in ("alpha", "lam", "iters", "cg", "applies", "slices", "r", "batch") if k in c},
            "parallelism": f"{par} x{world}"}


def quick_config_line(name, world, rank, local, torch, T, peak, flush, steps=3, warmup=3):
    """A short device-timed measurement of another BASELINE config inside the default (c2) run, so
    that all five configs appear in the driver-recorded line (`other_configs`). Same timing rules:
    warm-up, L2 flushed between steps, CUDA events; no e2e / CPU arm (use `--config` for the full
    line of that config)."""
    c = dict(CONFIGS[name])
    wl = Workload(name, c, world, rank, local, torch)
    for _ in range(warmup):
        wl.step()
    torch.cuda.synchronize()
    l0 = T.kernel_launches()
    r0 = wl.replayed_launches
    ms = 0.0
    for _ in range(steps):
        flush_l2(torch, flush)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        wl.step()
        e1.record()
        e1.synchronize()
        ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    launches = T.kernel_launches() - l0 + (wl.replayed_launches - r0)
    value = wl.units_per_step * steps / (ms * 1e-3)
    out = {"metric": c["metric"], "value": value, "unit": c["unit"], "ms_per_step": ms / steps, "steps": steps,
           "warmup": warmup, "dtype": c["prec"], "config": config_dict(name, c, world), "gpu_launches": int(launches)}
    k = c["kind"]
    if k != "sb_sur":
        applies = {"sb": c.get("iters", 1) * (c.get("cg", 0) + 1) * wl.units_per_step,
                   "cp": wl.units_per_step, "c1": wl.units_per_step, "apply": wl.units_per_step}[k]
        per_apply = apply_bytes(c, wl.op.info.wt_rows, complex_io=(k == "apply"), B=1)
        gbs = per_apply * applies * steps / (ms * 1e-3) / 1e9
        out["apply_in_step"] = {"bytes_per_apply": int(per_apply), "achieved": round(gbs, 1), "peak": peak,
                                "unit": "GB/s", "frac": round(gbs / peak, 4)}
    wl.op.close()
    del wl
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=0,
                    help="c1/c3: independent inputs per apply call; c2: slices solved per step (0: config)")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="default (c2) run: skip the short c1/c3/c4/c5 measurements reported in `other_configs`")
    ap.add_argument("--slices", type=int, default=0,
                    help="c4: total slices (0: config's 256); e.g. 32 on one GPU = one rank's share at N=8")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    if args.batch:
        c["batch"] = args.batch
    if args.slices:
        c["slices"] = args.slices
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (what the driver does itself)
        sys.exit(subprocess.call(launcher_cmd(args.gpus, sys.argv[1:])))
    if args.impl == "reference":
        # the reference's own CPU path on this box's host cores (rank 0 only; the other ranks
        # exit without work and without joining a process group)
        if int(os.environ.get("RANK", "0")) != 0:
            return
        cb = CpuBaseline(c)
        vals, walls = [], []
        for i in range(args.warmup + args.steps):
            v, wall, _ = cb.step()
            if i >= args.warmup:
                vals.append(v)
                walls.append(wall)
        cb.close()
        v = statistics.median(vals)
        line = {"impl": "reference", "metric": c["metric"], "value": v, "unit": c["unit"], "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                # one step = one concurrent bounded sample on every worker (wall time, measured)
                "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
                "scaling": scaling_of(c, args.gpus), "vs_baseline": None, "dtype": "f64",
                "data": DATA, "config": config_dict(args.config, c, args.gpus),
                "cpu_baseline": {"value": v, "unit": c["unit"], "cores": cb.cores, "kind": cb.kind,
                                 "sample": cb.describe(), "cpu_model": cb.model, "nproc": host_cpu()[1],
                                 "samples_per_step": cb.workers},
                "e2e": {"value": v, "unit": c["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    world, rank, local = dist_init()
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)
    import torch
    torch.cuda.set_device(local)
    import paper_1705_07497_b200 as T
    peak, peak_src = peaks()
    wl = Workload(args.config, c, world, rank, local, torch)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident in HBM, L2 flushed between steps)
    barrier(world)
    torch.cuda.synchronize()
    launches0 = T.kernel_launches()
    replayed0 = wl.replayed_launches
    total_ms = 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(torch, flush)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            wl.step()
            e1.record()
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    barrier(world)
    launches = T.kernel_launches() - launches0 + (wl.replayed_launches - replayed0)
    t_max = allreduce_max(total_ms, world)
    # sharded c5: all ranks work on the same applies (one slice) -> count them once
    units = float(wl.units_per_step * args.steps) if wl.sharded else allreduce_sum(float(wl.units_per_step * args.steps), world)
    launches = int(allreduce_sum(float(launches), world))
    value = units / (t_max * 1e-3)

    # ---- end to end through the C ABI with pinned host buffers
    wl.step_e2e()
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = 0.0
    for _ in range(max(1, min(args.steps, 3))):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        wl.step_e2e()
        e1.record()
        e1.synchronize()
        e2e_ms += max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3)
    e2e_steps = max(1, min(args.steps, 3))
    e2e_max = allreduce_max(e2e_ms, world)
    e2e_units = float(wl.units_per_step * e2e_steps) if wl.sharded else allreduce_sum(float(wl.units_per_step * e2e_steps), world)
    e2e_value = e2e_units / (e2e_max * 1e-3)

    top, roof = wl.roofline(peak)
    roof["peak_source"] = peak_src
    if "apply" in roof:
        # the same bytes per apply over the whole timed step (all kernels, launch gaps, lanes)
        k = c["kind"]
        applies = {"sb": c.get("iters", 1) * (c.get("cg", 0) + 1) * wl.units_per_step,
                   "cp": wl.units_per_step, "c1": wl.units_per_step, "apply": wl.units_per_step}[k]
        per_apply = apply_bytes(c, wl.op.info.wt_rows, complex_io=(k == "apply"), B=1)
        gbs = per_apply * applies * args.steps / (t_max * 1e-3) / 1e9
        roof["apply"]["in_step"] = {"applies_per_step": applies, "bytes_per_apply": int(per_apply),
                                    "achieved": round(gbs, 1), "frac": round(gbs / peak, 4)}
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file)).get(args.config, {}).get(top)
            if tr:
                roof["traffic"] = tr
        except Exception:
            pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = CpuBaseline(c)
        cb.step()  # worker start-up + operator construction (untimed)
        v, wall, _ = cb.step()
        cb.close()
        cpu = {"value": v, "unit": c["unit"], "cores": cb.cores, "kind": cb.kind, "sample": cb.describe(),
               "cpu_model": cb.model, "nproc": host_cpu()[1], "sample_wall_s": round(wall, 2)}

    info = wl.op.info
    h2d, d2h = int(wl.h2d), int(wl.d2h)
    others = None
    if world == 1 and args.config == "c2" and not args.no_other_configs and not args.batch:
        # the other four BASELINE configs, briefly, in the same run (device-timed values only)
        wl.op.close()
        del wl
        torch.cuda.empty_cache()
        others = {}
        for name in ("c1", "c3", "c4", "c5"):
            try:
                others[name] = quick_config_line(name, world, rank, local, torch, T, peak, flush)
            except Exception as e:  # never lose the headline line to a side measurement
                others[name] = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": c["metric"], "value": value, "unit": c["unit"], "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": scaling_of(c, world), "vs_baseline": None,
            "dtype": c["prec"], "data": DATA, "config": config_dict(args.config, c, world),
            "l2": "flushed between timed steps (256 MiB write)",
            "operator": {"wt_rows": int(info.wt_rows), "wt_slots": int(info.wt_slots), "P_local": int(info.P),
                         "nnz_local": int(info.nnz)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": c["unit"], "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if others is not None:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
