"""Benchmark suites and run driver of the reference (proj/src/bench.cpp, proj/include/tomo/bench.hpp)
on the B200 operators: RunConfig / describe / config_hash, prepare_run with the TOMOSPM1 operator
cache (load_or_build_sparse, bench.cpp:62-114), run_reconstruct, summarize (threshold crossings),
and the table1 / table2 / tables345 suites with the reference's CSV columns.

Differences from the reference, by design: times are CUDA-event times of the device solves
(time_apply: one warm-up, median of 5, like bench.cpp:245-257); the data noise is drawn with
numpy's seeded generator (the reference's default noise is 0, where both are identical);
reconstructions are written as .npy instead of PGM.
"""
from __future__ import annotations

import csv
import json
import math
import os
from dataclasses import dataclass, field, replace

import numpy as np

from . import tomo as T

PRESETS = {"digits2": 2, "digits6": 6, "digits12": 12}  # make_params (nufft.cpp:26-34)
BACKENDS = ("direct", "fused", "surrogate")


@dataclass
class RunConfig:
    """tomo::RunConfig (bench.hpp:10-31), same defaults."""

    n: int = 128
    d: int = 1
    preset: str = "digits6"
    backend: str = "fused"
    r: int = 1
    alpha: float = 1.0
    lambda_: float = 1.0
    iters: int = 200
    cg_steps: int = 5
    tol: float = 1e-8
    feedback: bool = False
    noise: float = 0.0
    seed: int = 0
    cache_dir: str = "cache"
    output_dir: str = "out"
    precision: str = "f64"  # B200 addition: operator / solver precision

    def validate(self):  # RunConfig::validate (bench.cpp:17-25)
        if self.n < 4 or self.n % 2:
            raise T.ConfigError("config: n must be even and >= 4")
        if self.d < 1:
            raise T.ConfigError("config: d must be >= 1")
        if self.backend == "surrogate" and not (1 <= self.r < self.n // 2):
            raise T.ConfigError("config: surrogate radius out of range")
        if self.noise < 0.0:
            raise T.ConfigError("config: negative noise")
        if self.preset not in PRESETS:
            raise T.ConfigError(f"unknown preset: {self.preset}")
        if self.backend not in BACKENDS:
            raise T.ConfigError(f"unknown backend: {self.backend}")

    def describe(self) -> str:
        """Canonical key=value line (bench.cpp:38-47; doubles as C++ ostream prints them)."""
        g = lambda v: f"{v:g}"  # noqa: E731
        return (f"n={self.n} d={self.d} preset={self.preset} backend={self.backend} r={self.r} "
                f"alpha={g(self.alpha)} lambda={g(self.lambda_)} iters={self.iters} cg_steps={self.cg_steps} "
                f"tol={g(self.tol)} feedback={1 if self.feedback else 0} noise={g(self.noise)} seed={self.seed}")

    def config_hash(self) -> str:
        """FNV-1a 64 of describe() (bench.cpp:49-58)."""
        h = 14695981039346656037
        for c in self.describe().encode():
            h ^= c
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return f"{h:016x}"

    def solver_config(self) -> T.SolverConfig:
        return T.SolverConfig(alpha=self.alpha, lambda_=self.lambda_, max_bregman_iters=self.iters,
                              cg_steps_per_update=self.cg_steps, update_tol_rel=self.tol,
                              data_feedback=self.feedback)


def geometry(c: RunConfig) -> T.Geometry:
    """make_angle_set(n, d) + slice_points + make_params(preset, n) (fourier_slice.cpp:10-41)."""
    count = int(math.floor(c.n * math.pi / (4.0 * c.d) + 0.5))
    if count < 2:
        raise T.ConfigError("make_angle_set: fewer than 2 angles")
    m_sp = PRESETS[c.preset]
    return T.Geometry(n=c.n, n_angles=count, win_lo=-m_sp, win_hi=m_sp, tau=m_sp / float(c.n * c.n))


def _cache_path(c: RunConfig, r: int) -> str:
    if r == 0:
        return os.path.join(c.cache_dir, f"btb_n{c.n}_{c.preset}_d{c.d}.tspm")
    return os.path.join(c.cache_dir, f"surrogate_n{c.n}_{c.preset}_d{c.d}_r{r}.tspm")


def _meta_matches(info: dict, c: RunConfig, g: T.Geometry, r: int) -> bool:
    return (info["n"] == c.n and info["m_sp"] == PRESETS[c.preset] and info["tau"] == g.tau
            and info["angle_count"] == g.n_angles and info["d"] == c.d and info["r"] == r)


def load_or_build(c: RunConfig, g: T.Geometry, log=None, **kw) -> T.NormalBackend:
    """load_or_build_sparse (bench.cpp:78-114) over the B200 backends; direct has no cache."""
    if c.backend == "direct":
        return T.make_direct_backend(g, precision=c.precision, **kw)
    r = 0 if c.backend == "fused" else c.r
    path = _cache_path(c, r)
    if os.path.exists(path):
        try:
            if _meta_matches(T.load_sparse_info(path), c, g, r):
                if log:
                    log(f"cached: {path}")
                return T.NormalBackend(g, c.backend, precision=c.precision, tspm=path, **kw)
            if log:
                log(f"cache metadata mismatch, rebuilding: {path}")
        except T.IoError as e:
            if log:
                log(f"cache unreadable ({e}), rebuilding: {path}")
    if c.backend == "fused":
        op = T.make_fused_backend(g, precision=c.precision, **kw)
    else:
        op = T.make_surrogate_backend(g, radius_r=c.r, precision=c.precision, **kw)
    os.makedirs(c.cache_dir, exist_ok=True)
    op.save_sparse(path, angle_subsample_d=c.d)
    if log:
        log(f"built and cached: {path}")
    return op


@dataclass
class RunSetup:
    geom: T.Geometry
    backend: T.NormalBackend
    phantom: np.ndarray
    data: np.ndarray


def prepare_run(c: RunConfig, log=None) -> RunSetup:
    """prepare_run (bench.cpp:118-150): Shepp-Logan phantom, data = F_NU^* phantom + noise."""
    c.validate()
    g = geometry(c)
    op = load_or_build(c, g, log)
    phantom = T.generate_shepp_logan(c.n)
    data = np.asarray(op.forward(phantom.astype(np.complex128 if op.f64 else np.complex64))).reshape(-1)
    if c.noise > 0.0:
        rng = np.random.default_rng(c.seed)
        data = data + c.noise * (rng.standard_normal(data.shape) + 1j * rng.standard_normal(data.shape))
    return RunSetup(g, op, phantom, data)


def precompute(c: RunConfig, log=None) -> list:
    """precompute (bench.cpp:152-171): build and cache the Gram (and the surrogate T)."""
    c.validate()
    g = geometry(c)
    paths = []
    load_or_build(replace(c, backend="fused"), g, log)
    paths.append(_cache_path(c, 0))
    if c.backend == "surrogate" or c.r >= 1:
        load_or_build(replace(c, backend="surrogate"), g, log)
        paths.append(_cache_path(c, c.r))
    return paths


@dataclass
class RunSummary:
    """tomo::RunSummary (bench.hpp:50-60)."""

    config: RunConfig
    iterations: int = 0
    total_s: float = 0.0
    cg_s: float = 0.0
    final_rel_l1: float = 0.0
    stopping_reason: str = ""
    threshold_crossings: list = field(default_factory=list)


THRESHOLDS = (1e-2, 1e-4, 1e-6, 1e-8)
THRESHOLD_NAMES = ("1e-2", "1e-4", "1e-6", "1e-8")


def summarize(c: RunConfig, trace: T.SolveTrace) -> RunSummary:
    """summarize (bench.cpp:173-194): first iteration with update < thr * first update."""
    s = RunSummary(c, trace.iterations, float(trace.t_total_s[-1]) if len(trace.t_total_s) else 0.0,
                   float(trace.t_cg_s[-1]) if len(trace.t_cg_s) else 0.0,
                   float(trace.rel_l1_err[-1]) if len(trace.rel_l1_err) else 0.0, trace.stopping_reason)
    for thr in THRESHOLDS:
        it, t = -1, -1.0
        for i, u in enumerate(trace.update_l1):
            if u < thr * trace.first_update_l1:
                it, t = i + 1, float(trace.t_total_s[i])
                break
        s.threshold_crossings.append((it, t))
    return s


def append_summary_jsonl(s: RunSummary, path: str):
    """append_summary_jsonl (bench.cpp:215-236)."""
    j = {"config": s.config.describe(), "config_hash": s.config.config_hash(), "iterations": s.iterations,
         "total_s": s.total_s, "cg_s": s.cg_s, "final_rel_l1": s.final_rel_l1, "stopping_reason": s.stopping_reason,
         "thresholds": [{"threshold": nm, "iteration": it, "seconds": t}
                        for nm, (it, t) in zip(THRESHOLD_NAMES, s.threshold_crossings)]}
    with open(path, "a") as f:
        f.write(json.dumps(j) + "\n")


def run_reconstruct(c: RunConfig, log=None):
    """run_reconstruct (bench.cpp:196-213): solve with the phantom as record_reference; writes
    recon_<hash>.npy, the trace CSV and a runs.jsonl line under output_dir."""
    setup = prepare_run(c, log)
    mu, traces = setup.backend.split_bregman_record(setup.data, c.solver_config(), reference=setup.phantom)
    trace = traces[0]
    os.makedirs(c.output_dir, exist_ok=True)
    stem = os.path.join(c.output_dir, "recon_" + c.config_hash())
    np.save(stem + ".npy", np.asarray(mu).reshape(c.n, c.n))
    trace.write_csv(stem + "_trace.csv")
    s = summarize(c, trace)
    append_summary_jsonl(s, os.path.join(c.output_dir, "runs.jsonl"))
    if log:
        log(f"run {c.config_hash()}: iters={s.iterations} rel_l1={s.final_rel_l1:g} reason={s.stopping_reason} "
            f"sigma={trace.stabilization_shift:g} min_ritz={trace.min_ritz:g}")
    return s, trace, mu


def scale_sizes(scale: str):
    if scale == "ci":  # B200 addition: the smallest sizes, for tests
        return [32, 64]
    if scale == "desk":
        return [64, 128]
    if scale == "paper":
        return [128, 256, 512]
    raise T.ConfigError("unknown scale: " + scale)


def time_apply(op: T.NormalBackend, probe, min_reps: int = 5) -> float:
    """time_apply (bench.cpp:245-257): one untimed warm-up, median of min_reps; CUDA events."""
    import torch
    x = torch.from_numpy(probe).cuda()
    op.apply_normal(x)
    times = []
    for _ in range(min_reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply_normal(x)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    return sorted(times)[len(times) // 2]


def bench_table1(scale: str, base: RunConfig, log) -> bool:
    """Per-apply time of the three backends (bench.cpp:259-297)."""
    ok = True
    with open(os.path.join(base.output_dir, f"table1_{scale}.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["config_hash", "n", "preset", "backend", "r", "apply_ms"])
        for n in scale_sizes(scale):
            for p in PRESETS:
                c = replace(base, n=n, preset=p)
                rng = np.random.default_rng(c.seed)
                probe = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
                for k in BACKENDS:
                    c = replace(c, backend=k)
                    try:
                        setup = prepare_run(c, log)
                        pr = probe.astype(np.complex128 if setup.backend.f64 else np.complex64)
                        ms = 1e3 * time_apply(setup.backend, pr, 5)
                        w.writerow([c.config_hash(), n, p, k, c.r if k == "surrogate" else 0, f"{ms:g}"])
                        log(f"table1 {n} {p} {k}: {ms:g} ms/apply")
                    except T.Error as e:
                        w.writerow([c.config_hash(), n, p, k, "", ""])
                        log(f"table1 row failed: {e}")
                        ok = False
    return ok


def bench_table2(scale: str, base: RunConfig, log) -> bool:
    """Fixed-iteration reconstructions (bench.cpp:299-326)."""
    ok = True
    with open(os.path.join(base.output_dir, f"table2_{scale}.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["config_hash", "n", "preset", "backend", "r", "iterations", "total_s", "cg_s", "final_rel_l1"])
        for n in scale_sizes(scale):
            for p in PRESETS:
                for k in BACKENDS:
                    c = replace(base, n=n, preset=p, backend=k, tol=0.0)
                    try:
                        s, _, _ = run_reconstruct(c, log)
                        w.writerow([c.config_hash(), n, p, k, c.r if k == "surrogate" else 0, s.iterations,
                                    f"{s.total_s:g}", f"{s.cg_s:g}", f"{s.final_rel_l1:g}"])
                    except T.Error as e:
                        log(f"table2 row failed: {e}")
                        ok = False
    return ok


def bench_tables345(scale: str, base: RunConfig, log) -> bool:
    """Tolerance runs with threshold crossings, d in {1, 2, 4} (bench.cpp:328-365)."""
    ok = True
    n = scale_sizes(scale)[-1]
    with open(os.path.join(base.output_dir, f"tables345_{scale}.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["config_hash", "n", "d", "backend", "r", "threshold", "iterations", "seconds",
                    "rel_l1_at_threshold"])
        for d in (1, 2, 4):
            for k in ("fused", "surrogate"):
                c = replace(base, n=n, d=d, backend=k, r=3, tol=1e-8)
                try:
                    setup = prepare_run(c, log)
                    _, traces = setup.backend.split_bregman_record(setup.data, c.solver_config(),
                                                                   reference=setup.phantom)
                    tr = traces[0]
                    s = summarize(c, tr)
                    for nm, (it, secs) in zip(THRESHOLD_NAMES, s.threshold_crossings):
                        w.writerow([c.config_hash(), n, d, k, c.r, nm, it, f"{secs:g}",
                                    f"{tr.rel_l1_err[it - 1]:g}" if it > 0 else "-1"])
                    tr.write_csv(os.path.join(base.output_dir, f"tables345_trace_{c.config_hash()}.csv"))
                except T.Error as e:
                    log(f"tables345 row failed: {e}")
                    ok = False
    return ok


def run_bench_suite(suite: str, scale: str, base: RunConfig, log=print) -> bool:
    """run_bench_suite (bench.cpp:369-382)."""
    os.makedirs(base.output_dir, exist_ok=True)
    if suite == "table1":
        return bench_table1(scale, base, log)
    if suite == "table2":
        return bench_table2(scale, base, log)
    if suite == "tables345":
        return bench_tables345(scale, base, log)
    if suite == "all":
        a = bench_table1(scale, base, log)
        b = bench_table2(scale, base, log)
        c = bench_tables345(scale, base, log)
        return a and b and c
    raise T.ConfigError("unknown suite: " + suite)
