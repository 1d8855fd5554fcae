"""ctypes binding of the CPU fp64 oracle (oracle/liboracle.so). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module; the product package never does. Every function here forwards to the C++
restatement in oracle/oracle.cpp, which cites the reference file:line it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class Geom(C.Structure):
    _fields_ = [("n", C.c_int), ("n_angles", C.c_int), ("n_b", C.c_int), ("oversample", C.c_int),
                ("win_lo", C.c_int), ("win_hi", C.c_int), ("tau", C.c_double),
                ("angles", C.POINTER(C.c_double))]


class System(C.Structure):
    _fields_ = [("backend", C.c_int), ("surrogate_r", C.c_int), ("euclidean", C.c_int),
                ("alpha", C.c_double), ("lambda_", C.c_double), ("shift", C.c_double),
                ("identity_k", C.c_int)]


class CgStats(C.Structure):
    _fields_ = [("steps_run", C.c_int), ("min_ritz", C.c_double), ("final_rs", C.c_double)]


class SbConfig(C.Structure):
    _fields_ = [("backend", C.c_int), ("surrogate_r", C.c_int), ("euclidean", C.c_int),
                ("alpha", C.c_double), ("lambda_", C.c_double), ("max_iters", C.c_int),
                ("cg_steps", C.c_int), ("update_tol_rel", C.c_double), ("warm_start", C.c_int),
                ("sigma_override", C.c_double), ("data_feedback", C.c_int)]


class SbTrace(C.Structure):
    _fields_ = [("iterations", C.c_int), ("first_update_l1", C.c_double), ("sigma", C.c_double),
                ("min_ritz", C.c_double), ("imag_leakage", C.c_double),
                ("stopped_on_tolerance", C.c_int)]


class CpConfig(C.Structure):
    _fields_ = [("alpha", C.c_double), ("lambda_", C.c_double), ("tau_cp", C.c_double),
                ("sigma_cp", C.c_double), ("theta", C.c_double), ("iters", C.c_int),
                ("cg_steps", C.c_int)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
        _LIB = C.CDLL(path)
        _LIB.orc_last_error.restype = C.c_char_p
        _LIB.orc_num_points.restype = C.c_int64
        _LIB.orc_btb_nnz.restype = C.c_int64
        _LIB.orc_rel_l1.restype = C.c_double
        _LIB.orc_rel_l1.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
        _LIB.orc_shrink.argtypes = [C.c_int64, C.c_void_p, C.c_double, C.c_void_p]
        _LIB.orc_random_ellipses.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        _LIB.orc_synthesize.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_uint64, C.c_void_p,
                                        C.c_void_p]
        _LIB.orc_lanczos_extreme.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_int,
                                             C.c_void_p]
        _LIB.orc_surrogate_sigma.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                             C.c_void_p]
        _LIB.orc_backproject.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        _LIB.orc_tikhonov_identity.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_int,
                                               C.c_double, C.c_void_p]
        _LIB.orc_cg.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_double, C.c_void_p, C.c_void_p]
    return _LIB


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Geometry:
    """Mirror of the geometry descriptor shared by the oracle and the product.

    Defaults reproduce the reference: n_b = n, R = 2, window [-m_sp, m_sp], tau = m_sp/n^2.
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
            self.tau = m_sp / float(self.n * self.n)

    @property
    def m(self):
        return self.oversample * self.n

    @property
    def P(self):
        return self.n_angles * self.n_b

    @property
    def w(self):
        return self.win_hi - self.win_lo + 1

    def cstruct(self) -> Geom:
        g = Geom(self.n, self.n_angles, self.n_b, self.oversample, self.win_lo, self.win_hi,
                 self.tau, None)
        if self.angles is not None:
            self._ang = _f64(self.angles)
            g.angles = self._ang.ctypes.data_as(C.POINTER(C.c_double))
        return g


def _g(geom: Geometry):
    s = geom.cstruct()
    return s, C.byref(s)


def points(geom):
    s, ref = _g(geom)
    out = np.empty((geom.P, 2))
    _check(lib().orc_points(ref, _p(out)))
    return out


def plan(geom):
    s, ref = _g(geom)
    near = np.empty((geom.P, 2), dtype=np.int32)
    e1 = np.empty((geom.P, 2))
    e2 = np.empty((geom.P, 2))
    e3 = np.empty(geom.w)
    _check(lib().orc_plan(ref, _p(near), _p(e1), _p(e2), _p(e3)))
    return near, e1, e2, e3


def weights(geom):
    s, ref = _g(geom)
    wx = np.empty((geom.P, geom.w))
    wy = np.empty((geom.P, geom.w))
    _check(lib().orc_weights(ref, _p(wx), _p(wy)))
    return wx, wy


def deapod(geom):
    s, ref = _g(geom)
    a = np.empty(geom.n)
    _check(lib().orc_deapod(ref, _p(a)))
    return a


def fft2(grid, inverse=False):
    g = _c128(grid).copy()
    m = g.shape[0]
    _check(lib().orc_fft2(C.c_int(m), _p(g), C.c_int(1 if inverse else 0)))
    return g


def interpolate(geom, grid):
    s, ref = _g(geom)
    gr = _c128(grid).reshape(-1)
    out = np.empty(geom.P, np.complex128)
    _check(lib().orc_interpolate(ref, _p(gr), _p(out)))
    return out


def spread(geom, samples):
    s, ref = _g(geom)
    sm = _c128(samples)
    out = np.empty(geom.m * geom.m, np.complex128)
    _check(lib().orc_spread(ref, _p(sm), _p(out)))
    return out.reshape(geom.m, geom.m)


def type2(geom, coeffs):
    s, ref = _g(geom)
    c = _c128(coeffs).reshape(-1)
    out = np.empty(geom.P, np.complex128)
    _check(lib().orc_type2(ref, _p(c), _p(out)))
    return out


def type1(geom, samples):
    s, ref = _g(geom)
    sm = _c128(samples)
    out = np.empty(geom.n * geom.n, np.complex128)
    _check(lib().orc_type1(ref, _p(sm), _p(out)))
    return out.reshape(geom.n, geom.n)


def direct_ndft(geom, data, to_type1):
    s, ref = _g(geom)
    d = _c128(data).reshape(-1)
    out = np.empty(geom.n * geom.n if to_type1 else geom.P, np.complex128)
    _check(lib().orc_direct_ndft(ref, _p(d), _p(out), C.c_int(1 if to_type1 else 0)))
    return out


def apply_normal(geom, u):
    s, ref = _g(geom)
    c = _c128(u).reshape(-1)
    out = np.empty_like(c)
    _check(lib().orc_apply_normal(ref, _p(c), _p(out)))
    return out.reshape(geom.n, geom.n)


def apply_normal_real(geom, u):
    s, ref = _g(geom)
    c = _f64(u).reshape(-1)
    out = np.empty_like(c)
    _check(lib().orc_apply_normal_real(ref, _p(c), _p(out)))
    return out.reshape(geom.n, geom.n)


def apply_normal_fused(geom, u):
    s, ref = _g(geom)
    c = _c128(u).reshape(-1)
    out = np.empty_like(c)
    _check(lib().orc_apply_normal_fused(ref, _p(c), _p(out)))
    return out.reshape(geom.n, geom.n)


def btb_nnz(geom):
    s, ref = _g(geom)
    v = lib().orc_btb_nnz(ref)
    if v < 0:
        _check(int(-v))
    return int(v)


def radial_weights(geom):
    s, ref = _g(geom)
    out = np.empty(geom.P)
    _check(lib().orc_radial_weights(ref, _p(out)))
    return out


def weighted_normal_real(geom, w, u):
    s, ref = _g(geom)
    ww = _f64(w)
    uu = _f64(u).reshape(-1)
    out = np.empty_like(uu)
    _check(lib().orc_weighted_normal_real(ref, _p(ww), _p(uu), _p(out)))
    return out.reshape(geom.n, geom.n)


def surrogate_stencil(geom, r):
    s, ref = _g(geom)
    out = np.empty((2 * r + 1) ** 2)
    _check(lib().orc_surrogate_stencil(ref, C.c_int(r), _p(out)))
    return out.reshape(2 * r + 1, 2 * r + 1)


def apply_stencil(n, r, stencil, u, euclidean=False):
    st = _f64(stencil).reshape(-1)
    uu = _f64(u).reshape(-1)
    out = np.empty_like(uu)
    _check(lib().orc_apply_stencil(C.c_int(n), C.c_int(r), C.c_int(int(euclidean)), _p(st), _p(uu),
                                   _p(out)))
    return out.reshape(n, n)


def grad(u):
    uu = _f64(u)
    n = uu.shape[0]
    gx = np.empty_like(uu)
    gy = np.empty_like(uu)
    _check(lib().orc_grad(C.c_int(n), _p(uu), _p(gx), _p(gy)))
    return gx, gy


def grad_adjoint(gx, gy):
    a = _f64(gx)
    b = _f64(gy)
    out = np.empty_like(a)
    _check(lib().orc_grad_adjoint(C.c_int(a.shape[0]), _p(a), _p(b), _p(out)))
    return out


def shrink(x, gamma):
    xx = _f64(x)
    out = np.empty_like(xx)
    _check(lib().orc_shrink(xx.size, _p(xx), gamma, _p(out)))
    return out


def system(backend=0, alpha=1.0, lam=1.0, shift=0.0, identity_k=False, r=1, euclidean=False):
    return System(backend, r, int(euclidean), alpha, lam, shift, int(identity_k))


def system_apply(geom, sysd: System, u):
    s, ref = _g(geom)
    uu = _f64(u).reshape(-1)
    out = np.empty_like(uu)
    _check(lib().orc_system_apply(ref, C.byref(sysd), _p(uu), _p(out)))
    return out.reshape(geom.n, geom.n)


def cg(geom, sysd: System, rhs, x0=None, steps=5, rel_tol=0.0):
    s, ref = _g(geom)
    b = _f64(rhs).reshape(-1)
    x0a = _f64(x0).reshape(-1) if x0 is not None else np.zeros_like(b)
    x = np.empty_like(b)
    st = CgStats()
    _check(lib().orc_cg(ref, C.byref(sysd), _p(b), _p(x0a), steps, rel_tol, _p(x), C.byref(st)))
    return x.reshape(geom.n, geom.n), st


def surrogate_sigma(geom, r, alpha, lam, euclidean=False):
    s, ref = _g(geom)
    out = C.c_double()
    _check(lib().orc_surrogate_sigma(ref, r, int(euclidean), alpha, lam, C.byref(out)))
    return out.value


def lanczos_extreme(geom, sysd, iters=40, seed=7, largest=False):
    s, ref = _g(geom)
    out = C.c_double()
    _check(lib().orc_lanczos_extreme(ref, C.byref(sysd), iters, seed, int(largest), C.byref(out)))
    return out.value


def backproject(geom, backend, alpha, f):
    s, ref = _g(geom)
    ff = _c128(f)
    out = np.empty(geom.n * geom.n)
    _check(lib().orc_backproject(ref, backend, alpha, _p(ff), _p(out)))
    return out.reshape(geom.n, geom.n)


def split_bregman(geom, f, backend=0, alpha=1.0, lam=1.0, max_iters=10, cg_steps=5,
                  update_tol_rel=0.0, warm_start=True, r=1, euclidean=False, sigma=None, feedback=False):
    s, ref = _g(geom)
    cfg = SbConfig(backend, r, int(euclidean), alpha, lam, max_iters, cg_steps, update_tol_rel,
                   int(warm_start), -1.0 if sigma is None else float(sigma), int(feedback))
    ff = _c128(f)
    mu = np.empty(geom.n * geom.n)
    upd = np.zeros(max_iters)
    tr = SbTrace()
    _check(lib().orc_split_bregman(ref, C.byref(cfg), _p(ff), _p(mu), _p(upd), C.byref(tr)))
    return mu.reshape(geom.n, geom.n), upd[:tr.iterations], tr


def tikhonov_identity(geom, f, alpha=1.0, steps=20, rel_tol=0.0):
    s, ref = _g(geom)
    ff = _c128(f)
    mu = np.empty(geom.n * geom.n)
    _check(lib().orc_tikhonov_identity(ref, alpha, _p(ff), steps, rel_tol, _p(mu)))
    return mu.reshape(geom.n, geom.n)


def chambolle_pock(geom, f, alpha=1.0, lam=1.0, tau_cp=0.35, sigma_cp=0.35, theta=1.0, iters=5,
                   cg_steps=15):
    s, ref = _g(geom)
    cfg = CpConfig(alpha, lam, tau_cp, sigma_cp, theta, iters, cg_steps)
    ff = _c128(f)
    mu = np.empty(geom.n * geom.n)
    _check(lib().orc_chambolle_pock(ref, C.byref(cfg), _p(ff), _p(mu)))
    return mu.reshape(geom.n, geom.n)


def shepp_logan(n):
    out = np.empty((n, n))
    _check(lib().orc_shepp_logan(C.c_int(n), _p(out)))
    return out


def random_ellipses(n, count=10, seed=0):
    out = np.empty((n, n))
    _check(lib().orc_random_ellipses(n, count, seed, _p(out)))
    return out


def synthesize(geom, phantom, noise_frac=0.0, seed=0):
    s, ref = _g(geom)
    ph = _f64(phantom).reshape(-1)
    out = np.empty(geom.P, np.complex128)
    sig = C.c_double()
    _check(lib().orc_synthesize(ref, _p(ph), noise_frac, seed, _p(out), C.byref(sig)))
    return out, sig.value


def set_perturbation(eps=0.0, seed=1):
    """Sensitivity probe: every real normal-operator input and output * (1 + eps N(0,1)); 0 = off."""
    lib().orc_set_perturbation.argtypes = [C.c_double, C.c_uint64]
    lib().orc_set_perturbation(float(eps), int(seed))


def rel_l1(cand, ref_):
    a = _f64(cand).reshape(-1)
    b = _f64(ref_).reshape(-1)
    return lib().orc_rel_l1(a.size, _p(a), _p(b))
