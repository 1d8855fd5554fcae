"""Python mirror of the reference's operator / solver API (proj/include/tomo/*.hpp) over the
B200 C ABI (include/tomo_b200.h).

Names follow the reference: ``SliceTransform``-style geometry, ``make_direct_backend`` /
``make_fused_backend`` / ``make_surrogate_backend`` (normal_ops.hpp:35-39), ``apply_normal`` / ``apply_normal_real``
(normal_ops.hpp:65-69), ``cg_solve`` (solver.hpp:43), ``split_bregman_tv`` (solver.hpp:83),
``tikhonov_solve`` (solver.hpp:91), ``grad`` / ``grad_adjoint`` / ``shrink`` (solver.hpp:19-24).
Errors are raised as the reference's exception classes (errors.hpp:9-30).

Arrays: torch CUDA tensors are passed to the kernels zero-copy (the call is ordered on the
current torch stream); numpy arrays are host buffers that the library stages to the device
and back (synchronous). Results come back in the kind that was passed in.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib


class Error(RuntimeError):
    """tomo::Error"""


class ConfigError(Error):
    """tomo::ConfigError (CLI exit code 2)"""


class NumericalError(Error):
    """tomo::NumericalError (CLI exit code 3)"""


class IoError(Error):
    """tomo::IoError (CLI exit code 4)"""


class CudaError(Error):
    """CUDA / NCCL failure inside libtomo_b200 (no reference analogue)."""


_ERRS = {_lib.TOMO_ERR_CONFIG: ConfigError, _lib.TOMO_ERR_NUMERICAL: NumericalError,
         _lib.TOMO_ERR_IO: IoError, _lib.TOMO_ERR_CUDA: CudaError}


def _check(rc: int):
    if rc != 0:
        raise _ERRS.get(rc, Error)(_lib.last_error())


def _torch():
    import torch
    return torch


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _stream_ptr(x):
    if _is_torch(x) and x.is_cuda:
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    return C.c_void_p(0)


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ConfigError("tensor must be contiguous")
        return C.c_void_p(x.data_ptr())
    return x.ctypes.data_as(C.c_void_p)


def _np_dtype(complex_: bool, f64: bool):
    if complex_:
        return np.complex128 if f64 else np.complex64
    return np.float64 if f64 else np.float32


def _torch_dtype(complex_: bool, f64: bool):
    torch = _torch()
    if complex_:
        return torch.complex128 if f64 else torch.complex64
    return torch.float64 if f64 else torch.float32


def _as_input(x, complex_: bool, f64: bool = False):
    """Contiguous view of x in the op's element type (torch tensor or array-like)."""
    if _is_torch(x):
        want = _torch_dtype(complex_, f64)
        if x.dtype != want:
            x = x.to(want)
        return x.contiguous()
    return np.ascontiguousarray(x, dtype=_np_dtype(complex_, f64))


def _empty_like_kind(x, shape, complex_: bool, f64: bool = False):
    if _is_torch(x):
        torch = _torch()
        pin = (not x.is_cuda) and x.is_pinned()
        return torch.empty(shape, dtype=_torch_dtype(complex_, f64), device=x.device, pin_memory=pin)
    return np.empty(shape, dtype=_np_dtype(complex_, f64))


@dataclass
class Geometry:
    """SliceGrid + NufftParams (fourier_slice.hpp:24-28, nufft.hpp:16-21) with extensions.

    Defaults are the reference's: n_b = n, R = 2, window [-m_sp, m_sp], tau = m_sp/n^2,
    theta_a = a*pi/A.
    """

    n: int
    n_angles: int
    n_b: int = 0
    oversample: int = 2
    win_lo: int = -6
    win_hi: int = 6
    tau: float = 0.0
    angles: np.ndarray | None = None

    def __post_init__(self):
        if self.n_b == 0:
            self.n_b = self.n
        if self.tau == 0.0:
            m_sp = max(self.win_hi, -self.win_lo)
            if self.oversample == 2:
                self.tau = m_sp / float(self.n * self.n)  # nufft.cpp:33
            else:  # Greengard-Lee rule for R != 2 (extension D7)
                R = self.oversample
                self.tau = math.pi * m_sp / (self.n * self.n * R * (R - 0.5))

    @classmethod
    def from_preset(cls, n, n_angles, m_sp, **kw):
        return cls(n=n, n_angles=n_angles, win_lo=-m_sp, win_hi=m_sp, **kw)

    @property
    def m(self):
        return self.oversample * self.n

    @property
    def P(self):
        return self.n_angles * self.n_b

    @property
    def window(self):
        return self.win_hi - self.win_lo + 1

    def _desc(self):
        d = _lib.GeomDesc(self.n, self.n_angles, self.n_b, self.oversample, self.win_lo, self.win_hi, self.tau, None)
        if self.angles is not None:
            self._ang = np.ascontiguousarray(self.angles, dtype=np.float64)
            d.angles = self._ang.ctypes.data_as(C.POINTER(C.c_double))
        return d


@dataclass
class SolverConfig:
    """tomo::SolverConfig (solver.hpp:51-65)."""

    alpha: float = 1.0
    lambda_: float = 1.0
    max_bregman_iters: int = 6000
    cg_steps_per_update: int = 5
    update_tol_rel: float = 1e-8
    warm_start: bool = True
    sigma_override: float | None = None
    data_feedback: bool = False  # outer residual feedback on the data term (solver.hpp:58-61)


@dataclass
class SolveTrace:
    """tomo::SolveTrace (solver.hpp:67-80), one per slice."""

    update_l1: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterations: int = 0
    stopping_reason: str = "max_iterations"
    first_update_l1: float = 0.0
    stabilization_shift: float = 0.0
    min_ritz: float = 0.0
    imag_leakage: float = 0.0
    rel_l1_err: np.ndarray = field(default_factory=lambda: np.zeros(0))  # with record_reference
    t_total_s: np.ndarray = field(default_factory=lambda: np.zeros(0))   # recorded solves only
    t_cg_s: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def write_csv(self, path):
        """SolveTrace::write_csv (solver.cpp:140-150)."""
        with open(path, "w") as f:
            f.write("iter,update_l1,rel_l1_err,t_total_s,t_cg_s\n")
            for i, u in enumerate(self.update_l1):
                rel = f"{self.rel_l1_err[i]:.6g}" if i < len(self.rel_l1_err) else ""
                tt = self.t_total_s[i] if i < len(self.t_total_s) else 0.0
                tc = self.t_cg_s[i] if i < len(self.t_cg_s) else 0.0
                f.write(f"{i + 1},{u:.6g},{rel},{tt:.6g},{tc:.6g}\n")


@dataclass
class CgStats:
    steps_run: int = 0
    min_ritz: float = 0.0
    final_rs: float = 0.0


class NormalBackend:
    """Device-resident normal operator (tomo::NormalBackend, normal_ops.hpp:23-31).

    kind "direct": N = F_NU F_NU^* through the precomputed W (SELL-32 ELL) and W^T tables and
    the pruned in-CTA FFT passes; kind "fused": the same FFT passes around one SpMV with the
    Gram W^T W (build_btb / apply_normal_fused, normal_ops.cpp:53-206); kind "surrogate": the
    translated stencil T.
    """

    _KINDS = {"direct": _lib.BACKEND_DIRECT, "fused": _lib.BACKEND_FUSED, "surrogate": _lib.BACKEND_SURROGATE}

    def __init__(self, geom: Geometry, kind: str = "direct", surrogate_r: int = 1, euclidean: bool = False,
                 device: int = 0, angle_block: tuple[int, int] | None = None, max_batch: int = 1,
                 precision: str = "f32", mem_cap_bytes: int = 0, tspm: str | None = None):
        if kind not in self._KINDS:
            raise ConfigError(f"unknown backend: {kind}")
        if precision not in ("f32", "f64"):
            raise ConfigError(f"unknown precision: {precision}")
        self.geom = geom
        self.kind = kind
        self.device = device
        self.precision = precision
        self.f64 = precision == "f64"
        ab = angle_block or (0, 0)
        desc = _lib.OpDesc(self._KINDS[kind], surrogate_r, int(euclidean), device, ab[0], ab[1], max_batch,
                           _lib.F64 if self.f64 else _lib.F32, int(mem_cap_bytes))
        gd = geom._desc()
        h = C.c_void_p()
        if tspm is not None:  # load_or_build_sparse's cached operator (bench.cpp:78-114)
            _check(lib().tomo_op_create_tspm(C.byref(gd), C.byref(desc), os.fsencode(tspm), C.byref(h)))
        else:
            _check(lib().tomo_op_create(C.byref(gd), C.byref(desc), C.byref(h)))
        self._h = h
        self._allreduce_cb = None

    def close(self):
        if getattr(self, "_h", None):
            lib().tomo_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- info
    @property
    def info(self) -> _lib.OpInfo:
        inf = _lib.OpInfo()
        _check(lib().tomo_op_get_info(self._h, C.byref(inf)))
        return inf

    def stencil(self) -> np.ndarray:
        inf = self.info
        r = inf.surrogate_r
        s = 2 * r + 1
        return np.array(inf.stencil[: s * s]).reshape(s, s)

    # ---------------------------------------------------------------- helpers
    def _batch(self, x, per_item: int):
        size = x.numel() if _is_torch(x) else x.size
        if size % per_item:
            raise ConfigError("input size is not a multiple of the per-slice size")
        return size // per_item

    def _unary(self, fn, x, in_complex, out_complex, in_items, out_shape_of):
        x = _as_input(x, in_complex, self.f64)
        B = self._batch(x, in_items)
        out = _empty_like_kind(x, out_shape_of(x, B), out_complex, self.f64)
        _check(fn(self._h, _ptr(x), _ptr(out), B, _stream_ptr(x)))
        return out

    def _img_shape(self, x, B):
        n = self.geom.n
        return tuple(x.shape) if (x.shape[-2:] == (n, n) if len(x.shape) >= 2 else False) else (B, n, n)

    # ---------------------------------------------------------------- operators
    def apply_normal(self, image):
        """apply_normal (normal_ops.hpp:65): complex64 (.., n, n) -> complex64."""
        n2 = self.geom.n ** 2
        return self._unary(lib().tomo_apply_normal, image, True, True, n2, self._img_shape)

    def apply_normal_real(self, u):
        """apply_normal_real (normal_ops.hpp:69): Re(N u), float32 (.., n, n)."""
        n2 = self.geom.n ** 2
        return self._unary(lib().tomo_apply_normal_real, u, False, False, n2, self._img_shape)

    def forward(self, image):
        """SliceTransform::forward — type-2 NUFFT onto the slice points (B, P)."""
        n2, P = self.geom.n ** 2, self.info.P
        return self._unary(lib().tomo_forward, image, True, True, n2, lambda x, B: (B, P))

    def forward_real(self, image):
        """forward_transform (fourier_slice.cpp:61-64): type-2 of a real image (B, P), through the
        Hermitian half grid."""
        n2, P = self.geom.n ** 2, self.info.P
        return self._unary(lib().tomo_forward_real, image, False, True, n2, lambda x, B: (B, P))

    def adjoint(self, samples):
        """SliceTransform::adjoint — type-1 NUFFT back to the image (B, n, n)."""
        P = self.info.P
        n = self.geom.n
        return self._unary(lib().tomo_adjoint, samples, True, True, P, lambda x, B: (B, n, n))

    def spmv_w(self, grid):
        """W (interpolate) on the internal grid layout node = iy*m + ix."""
        m, P = self.geom.m, self.info.P
        return self._unary(lib().tomo_spmv_w, grid, True, True, m * m, lambda x, B: (B, P))

    def spmv_wt(self, samples):
        """W^T (spread) onto the internal grid layout node = iy*m + ix."""
        m, P = self.geom.m, self.info.P
        return self._unary(lib().tomo_spmv_wt, samples, True, True, P, lambda x, B: (B, m, m))

    def backproject(self, slice_data, alpha=1.0, weighted=None):
        """make_subproblem backprojection (solver.cpp:200-213)."""
        if weighted is None:
            weighted = self.kind == "surrogate"
        f = _as_input(slice_data, True, self.f64)
        B = self._batch(f, self.info.P)
        n = self.geom.n
        out = _empty_like_kind(f, (B, n, n), False, self.f64)
        _check(lib().tomo_backproject(self._h, float(alpha), int(weighted), _ptr(f), _ptr(out), B, _stream_ptr(f)))
        return out

    # ---------------------------------------------------------------- solvers
    def cg(self, rhs, x0=None, alpha=1.0, lambda_=1.0, shift=0.0, steps=5, rel_tol=0.0):
        """cg_solve (solver.cpp:56-95) on alpha*B + lambda*K'K + shift*I; returns (x, [CgStats])."""
        b = _as_input(rhs, False, self.f64)
        n2 = self.geom.n ** 2
        B = self._batch(b, n2)
        x0c = _as_input(x0, False, self.f64) if x0 is not None else None
        x = _empty_like_kind(b, self._img_shape(b, B), False, self.f64)
        sysd = _lib.System(alpha, lambda_, shift)
        st = (_lib.CgStats * B)()
        _check(lib().tomo_cg(self._h, C.byref(sysd), _ptr(b), _ptr(x0c), _ptr(x), steps, rel_tol, B, st,
                             _stream_ptr(b)))
        return x, [CgStats(s.steps_run, s.min_ritz, s.final_rs) for s in st]

    def split_bregman(self, slice_data, config: SolverConfig):
        """split_bregman_tv (solver.cpp:219-307) on a batch of slices; returns (mu, [SolveTrace])."""
        f = _as_input(slice_data, True, self.f64)
        B = self._batch(f, self.info.P)
        n = self.geom.n
        mu = _empty_like_kind(f, (B, n, n), False, self.f64)
        cfg = _lib.SbConfig(config.alpha, config.lambda_, config.max_bregman_iters, config.cg_steps_per_update,
                            config.update_tol_rel, int(config.warm_start),
                            -1.0 if config.sigma_override is None else float(config.sigma_override),
                            int(config.data_feedback))
        upd = np.zeros(B * config.max_bregman_iters)
        tr = (_lib.SbTrace * B)()
        _check(lib().tomo_split_bregman(self._h, C.byref(cfg), _ptr(f), _ptr(mu), B,
                                        upd.ctypes.data_as(C.c_void_p), tr, _stream_ptr(f)))
        traces = []
        for b in range(B):
            t = tr[b]
            traces.append(SolveTrace(upd.reshape(B, -1)[b, : t.iterations].copy(), t.iterations,
                                     "tolerance" if t.stopped_on_tolerance else "max_iterations",
                                     t.first_update_l1, t.sigma, t.min_ritz, t.imag_leakage))
        return mu, traces

    def split_bregman_record(self, slice_data, config: SolverConfig, reference=None):
        """split_bregman_tv with the reference's per-iteration trace: t_total_s / t_cg_s (CUDA
        events, one graph launch per CG and per update) and, given the phantom(s) as
        `reference` (record_reference, solver.cpp:291-294), rel_l1_err per iteration."""
        f = _as_input(slice_data, True, self.f64)
        B = self._batch(f, self.info.P)
        n = self.geom.n
        mu = _empty_like_kind(f, (B, n, n), False, self.f64)
        ref = None
        if reference is not None:
            ref = _as_input(reference, False, self.f64)
            size = ref.size if isinstance(ref, np.ndarray) else ref.numel()
            if size != B * n * n:
                raise ConfigError("split_bregman_record: reference must hold batch x n^2 values")
        cfg = _lib.SbConfig(config.alpha, config.lambda_, config.max_bregman_iters, config.cg_steps_per_update,
                            config.update_tol_rel, int(config.warm_start),
                            -1.0 if config.sigma_override is None else float(config.sigma_override),
                            int(config.data_feedback))
        K = config.max_bregman_iters
        upd, rel = np.zeros(B * K), np.zeros(B * K)
        tt, tc = np.zeros(K), np.zeros(K)
        tr = (_lib.SbTrace * B)()
        vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _check(lib().tomo_split_bregman_record(self._h, C.byref(cfg), _ptr(f), _ptr(mu), B,
                                               _ptr(ref) if ref is not None else None, vp(upd),
                                               vp(rel) if ref is not None else None, vp(tt), vp(tc), tr,
                                               _stream_ptr(f)))
        traces = []
        for b in range(B):
            t = tr[b]
            k = t.iterations
            traces.append(SolveTrace(upd.reshape(B, K)[b, :k].copy(), k,
                                     "tolerance" if t.stopped_on_tolerance else "max_iterations",
                                     t.first_update_l1, t.sigma, t.min_ritz, t.imag_leakage,
                                     rel.reshape(B, K)[b, :k].copy() if ref is not None else np.zeros(0),
                                     tt[:k].copy(), tc[:k].copy()))
        return mu, traces

    def tikhonov(self, slice_data, alpha=1.0, steps=20, rel_tol=0.0):
        """Config-1 KKT solve: (alpha N + I) mu = alpha Re(F_NU f), fixed steps (solver.cpp:309-337)."""
        f = _as_input(slice_data, True, self.f64)
        B = self._batch(f, self.info.P)
        n = self.geom.n
        mu = _empty_like_kind(f, (B, n, n), False, self.f64)
        _check(lib().tomo_tikhonov(self._h, float(alpha), _ptr(f), _ptr(mu), steps, rel_tol, B, _stream_ptr(f)))
        return mu

    def chambolle_pock(self, slice_data, alpha=1.0, lambda_=1.0, tau_cp=0.35, sigma_cp=0.35, theta=1.0,
                       iters=10, cg_steps=15):
        """Chambolle-Pock anisotropic TV with CG primal prox (extension of PAPER.md:40-48)."""
        f = _as_input(slice_data, True, self.f64)
        B = self._batch(f, self.info.P)
        n = self.geom.n
        mu = _empty_like_kind(f, (B, n, n), False, self.f64)
        cfg = _lib.CpConfig(alpha, lambda_, tau_cp, sigma_cp, theta, iters, cg_steps)
        _check(lib().tomo_chambolle_pock(self._h, C.byref(cfg), _ptr(f), _ptr(mu), B, _stream_ptr(f)))
        return mu

    def profile_stages(self, batch=1, reps=20, complex_io=False):
        """Per-kernel device time (ms, CUDA events on the current stream) and algorithmic bytes
        of one hot-path solver step (complex_io: of one complex apply); {name: (ms, bytes)} for
        the stages this backend runs."""
        torch = _torch()
        ms = np.zeros(_lib.NUM_STAGES)
        by = np.zeros(_lib.NUM_STAGES)
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().tomo_profile_stages(self._h, batch, reps, int(bool(complex_io)), ms.ctypes.data_as(C.c_void_p),
                                         by.ctypes.data_as(C.c_void_p), stream))
        out = {name: (float(ms[i]), float(by[i])) for i, name in enumerate(_lib.STAGE_NAMES) if by[i] > 0}
        return out

    # ---------------------------------------------------------------- on-disk operators
    def save_sparse(self, path, angle_subsample_d: int = 1):
        """save_sparse (sparse.cpp:68-106) of the Gram (fused) or surrogate T, TOMOSPM1."""
        _check(lib().tomo_op_save_tspm(self._h, os.fsencode(path), int(angle_subsample_d)))

    # ---------------------------------------------------------------- multi-GPU
    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int):
        _check(lib().tomo_op_attach_nccl(self._h, unique_id, nranks, rank))

    def set_allreduce(self, fn):
        """fn(buf_ptr:int, count:int, stream_ptr:int) -> None, summing the op's element type in place."""
        def cb(buf, count, precision, stream, user):
            try:
                fn(buf, count, stream)
                return 0
            except Exception:  # pragma: no cover
                return 1
        self._allreduce_cb = _lib.ALLREDUCE_FN(cb)
        _check(lib().tomo_op_set_allreduce(self._h, self._allreduce_cb, None))


def load_sparse_info(path) -> dict:
    """load_sparse (sparse.cpp:108-141) + validate: header and provenance trailer of a TOMOSPM1 file."""
    m = _lib.TspmMeta()
    _check(lib().tomo_tspm_info(os.fsencode(path), C.byref(m)))
    return {k: getattr(m, k) for k, _ in m._fields_}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().tomo_nccl_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------- reference-named functions
def make_direct_backend(geom: Geometry, **kw) -> NormalBackend:
    return NormalBackend(geom, "direct", **kw)


def make_fused_backend(geom: Geometry, mem_cap_bytes: int = 8 << 30, **kw) -> NormalBackend:
    """make_fused_backend (normal_ops.hpp:37): Gram W^T W, refused above `mem_cap_bytes`."""
    return NormalBackend(geom, "fused", mem_cap_bytes=mem_cap_bytes, **kw)


def make_surrogate_backend(geom: Geometry, radius_r: int = 1, euclidean: bool = False, **kw) -> NormalBackend:
    return NormalBackend(geom, "surrogate", surrogate_r=radius_r, euclidean=euclidean, **kw)


def apply_normal(backend: NormalBackend, image):
    return backend.apply_normal(image)


def apply_normal_real(backend: NormalBackend, u):
    return backend.apply_normal_real(u)


def split_bregman_tv(backend: NormalBackend, slice_data, config: SolverConfig):
    mu, traces = backend.split_bregman(slice_data, config)
    return mu, traces


def tikhonov_solve(backend: NormalBackend, slice_data, alpha=1.0, steps=20, rel_tol=0.0):
    return backend.tikhonov(slice_data, alpha, steps, rel_tol)


def radial_density_weights(geom: Geometry) -> np.ndarray:
    """normal_ops.cpp:208-219: |k_r| per sample (DC: 1/4), angle-major."""
    kr = np.arange(geom.n_b) - geom.n_b // 2
    w = np.where(kr == 0, 0.25, np.abs(kr)).astype(np.float64)
    return np.tile(w, geom.n_angles)


def _prec_of(x):
    torch = _torch()
    if x.dtype == torch.float64:
        return _lib.F64, x.contiguous()
    return _lib.F32, x.contiguous().float()


def grad(u):
    """grad (solver.cpp:12-25) on a CUDA tensor (.., n, n), float32 or float64."""
    torch = _torch()
    prec, u = _prec_of(u)
    n = u.shape[-1]
    B = u.numel() // (n * n)
    gx, gy = torch.empty_like(u), torch.empty_like(u)
    _check(lib().tomo_grad(n, prec, _ptr(u), _ptr(gx), _ptr(gy), B, _stream_ptr(u)))
    return gx, gy


def grad_adjoint(gx, gy):
    torch = _torch()
    prec, gx = _prec_of(gx)
    gy = gy.contiguous().to(gx.dtype)
    n = gx.shape[-1]
    B = gx.numel() // (n * n)
    out = torch.empty_like(gx)
    _check(lib().tomo_grad_adjoint(n, prec, _ptr(gx), _ptr(gy), _ptr(out), B, _stream_ptr(gx)))
    return out


def shrink(x, gamma: float):
    torch = _torch()
    prec, x = _prec_of(x)
    out = torch.empty_like(x)
    _check(lib().tomo_shrink(x.numel(), prec, _ptr(x), float(gamma), _ptr(out), _stream_ptr(x)))
    return out


def generate_shepp_logan(n: int) -> np.ndarray:
    out = np.empty((n, n), np.float32)
    _check(lib().tomo_shepp_logan(n, out.ctypes.data_as(C.c_void_p)))
    return out


def random_ellipses(n: int, count: int = 10, seed: int = 0) -> np.ndarray:
    out = np.empty((n, n), np.float32)
    _check(lib().tomo_random_ellipses(n, count, seed, out.ctypes.data_as(C.c_void_p)))
    return out


def kernel_launches() -> int:
    return int(lib().tomo_kernel_launches())


def fft_rows(x, inverse=False):
    """Test hook: batched length-m FFT rows through the in-CTA Stockham kernel (unscaled)."""
    torch = _torch()
    f64 = x.dtype == torch.complex128
    x = x.contiguous().to(torch.complex128 if f64 else torch.complex64)
    rows, m = x.shape
    out = torch.empty_like(x)
    _check(lib().tomo_fft_rows(m, rows, _lib.F64 if f64 else _lib.F32, _ptr(x), _ptr(out), int(inverse),
                               _stream_ptr(x)))
    return out
