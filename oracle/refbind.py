"""ctypes binding of oracle/_ref/libtomo_ref.so — the reference's own sources built against the
Eigen-API shim (TEST INFRASTRUCTURE ONLY; see oracle/ref_driver.cpp and oracle/Makefile).

Used by tests/test_oracle_pin.py, tests/golden/make_golden.py and bench.py --impl reference.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_ref", "libtomo_ref.so")
_LIB = None


def _host_has_avx512() -> bool:
    """libtomo_ref.so is built with the reference's -march=native (Sapphire Rapids here; the GPU
    boxes are Emerald Rapids, same ISA): refuse it on a host without AVX-512F."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return "avx512f" in line.split()
    except OSError:
        pass
    return False


def available() -> bool:
    return os.path.exists(_PATH) and _host_has_avx512()


def lib():
    global _LIB
    if _LIB is None:
        _LIB = C.CDLL(_PATH)
        _LIB.ref_last_error.restype = C.c_char_p
        _LIB.ref_btb_nnz.restype = C.c_int64
        d = C.c_double
        _LIB.ref_points.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_void_p]
        for name in ("ref_type2", "ref_type1"):
            getattr(_LIB, name).argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_void_p, C.c_void_p]
        _LIB.ref_plan.argtypes = [C.c_int, C.c_int, C.c_int, d] + [C.c_void_p] * 4
        _LIB.ref_direct_ndft.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_void_p, C.c_void_p, C.c_int]
        for name in ("ref_apply_normal", "ref_apply_normal_real"):
            getattr(_LIB, name).argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_int, C.c_void_p, C.c_void_p]
        _LIB.ref_btb_nnz.argtypes = [C.c_int, C.c_int, C.c_int, d]
        _LIB.ref_surrogate_stencil.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_int, C.c_void_p]
        _LIB.ref_apply_surrogate_real.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_int, C.c_void_p,
                                                  C.c_void_p]
        _LIB.ref_cg_sb_system.argtypes = [C.c_int, C.c_int, C.c_int, d, d, d, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_void_p, C.c_void_p]
        _LIB.ref_split_bregman.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_int, C.c_int, d, d, C.c_int,
                                           C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p]
        _LIB.ref_tikhonov_identity.argtypes = [C.c_int, C.c_int, C.c_int, d, d, C.c_void_p, C.c_int,
                                               C.c_void_p]
        _LIB.ref_shepp_logan.argtypes = [C.c_int, C.c_void_p]
        _LIB.ref_set_nb.argtypes = [C.c_int]
        _LIB.ref_set_feedback.argtypes = [C.c_int]
        _LIB.ref_save_btb.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_char_p]
        _LIB.ref_save_surrogate.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_int, C.c_int, C.c_char_p]
        _LIB.ref_synthesize.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_void_p, d, C.c_uint64, C.c_void_p]
        _LIB.ref_backend_new.restype = C.c_void_p
        _LIB.ref_backend_new.argtypes = [C.c_int, C.c_int, C.c_int, d, C.c_int, C.c_int, C.c_int]
        _LIB.ref_backend_free.argtypes = [C.c_void_p]
        _LIB.ref_backend_time_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _LIB.ref_backend_split_bregman.argtypes = [C.c_void_p, d, d, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                                   C.c_void_p, C.c_void_p]
    return _LIB


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Ref:
    """Reference geometry: R = 2, window [-m_sp, m_sp], theta_a = a*pi/A; n_b radial samples
    (default n, the reference; other values go through the reference's FrequencyPointSet /
    SliceTransform with the slice_points lattice at spacing 2*pi/n_b)."""

    def __init__(self, n, n_angles, m_sp, tau=None, n_b=0):
        self.n, self.A, self.m_sp = n, n_angles, m_sp
        self.n_b = n_b or n
        self.tau = tau if tau is not None else m_sp / float(n * n)
        self.P = self.n_b * n_angles
        self._a = (n, n_angles, m_sp, self.tau)
        lib().ref_set_nb(self.n_b)

    def points(self):
        out = np.empty((self.P, 2))
        _check(lib().ref_points(*self._a, _p(out)))
        return out

    def plan(self):
        near = np.empty((self.P, 2), np.int32)
        e1 = np.empty((self.P, 2))
        e2 = np.empty((self.P, 2))
        e3 = np.empty(2 * self.m_sp + 1)
        _check(lib().ref_plan(*self._a, _p(near), _p(e1), _p(e2), _p(e3)))
        return near, e1, e2, e3

    def type2(self, u):
        u = np.ascontiguousarray(u, np.complex128)
        out = np.empty(self.P, np.complex128)
        _check(lib().ref_type2(*self._a, _p(u), _p(out)))
        return out

    def type1(self, s):
        s = np.ascontiguousarray(s, np.complex128)
        out = np.empty((self.n, self.n), np.complex128)
        _check(lib().ref_type1(*self._a, _p(s), _p(out)))
        return out

    def direct_ndft(self, x, to_type1):
        x = np.ascontiguousarray(x, np.complex128)
        out = np.empty(self.n * self.n if to_type1 else self.P, np.complex128)
        _check(lib().ref_direct_ndft(*self._a, _p(x), _p(out), int(to_type1)))
        return out

    def apply_normal(self, u, fused=False):
        u = np.ascontiguousarray(u, np.complex128)
        out = np.empty((self.n, self.n), np.complex128)
        _check(lib().ref_apply_normal(*self._a, int(fused), _p(u), _p(out)))
        return out

    def apply_normal_real(self, u, fused=False):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty((self.n, self.n))
        _check(lib().ref_apply_normal_real(*self._a, int(fused), _p(u), _p(out)))
        return out

    def btb_nnz(self):
        return int(lib().ref_btb_nnz(*self._a))

    def save_btb(self, path):
        """make_fused_backend + save_sparse: the reference's TOMOSPM1 Gram file."""
        _check(lib().ref_save_btb(*self._a, str(path).encode()))

    def save_surrogate(self, path, r, euclidean=False):
        """build_surrogate + save_sparse: the reference's TOMOSPM1 surrogate T file."""
        _check(lib().ref_save_surrogate(*self._a, r, int(euclidean), str(path).encode()))

    def surrogate_stencil(self, r):
        out = np.zeros((2 * r + 1, 2 * r + 1))
        _check(lib().ref_surrogate_stencil(*self._a, r, _p(out)))
        return out

    def apply_surrogate_real(self, r, u):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty((self.n, self.n))
        _check(lib().ref_apply_surrogate_real(*self._a, r, _p(u), _p(out)))
        return out

    def cg_sb_system(self, alpha, lam, rhs, x0=None, steps=5):
        rhs = np.ascontiguousarray(rhs, np.float64)
        x0 = np.zeros_like(rhs) if x0 is None else np.ascontiguousarray(x0, np.float64)
        x = np.empty_like(rhs)
        mr = C.c_double()
        _check(lib().ref_cg_sb_system(*self._a, alpha, lam, _p(rhs), _p(x0), steps, _p(x), C.byref(mr)))
        return x, mr.value

    def split_bregman(self, f, backend=0, r=1, alpha=1.0, lam=1.0, iters=5, cg_steps=5, feedback=False):
        f = np.ascontiguousarray(f, np.complex128)
        mu = np.empty((self.n, self.n))
        upd = np.empty(iters)
        sg = C.c_double()
        lk = C.c_double()
        lib().ref_set_feedback(int(feedback))
        try:
            _check(lib().ref_split_bregman(*self._a, backend, r, alpha, lam, iters, cg_steps, _p(f), _p(mu),
                                           _p(upd), C.byref(sg), C.byref(lk)))
        finally:
            lib().ref_set_feedback(0)
        return mu, upd, sg.value, lk.value

    def tikhonov_identity(self, f, alpha=1.0, steps=20):
        f = np.ascontiguousarray(f, np.complex128)
        mu = np.empty((self.n, self.n))
        _check(lib().ref_tikhonov_identity(*self._a, alpha, _p(f), steps, _p(mu)))
        return mu

    def synthesize(self, phantom, sigma, seed):
        ph = np.ascontiguousarray(phantom, np.float64)
        out = np.empty(self.P, np.complex128)
        _check(lib().ref_synthesize(*self._a, _p(ph), sigma, seed, _p(out)))
        return out


def shepp_logan(n):
    out = np.empty((n, n))
    _check(lib().ref_shepp_logan(n, _p(out)))
    return out


class RefBackend:
    """A reference NormalBackend built once (construction untimed) for timing the
    reference's own apply_normal (time_apply semantics, bench.cpp:245-257) and split_bregman_tv."""

    def __init__(self, n, n_angles, m_sp, tau=None, n_b=0, backend=0, r=1):
        self.n = n
        self.P = (n_b or n) * n_angles
        tau = tau if tau is not None else m_sp / float(n * n)
        self._h = lib().ref_backend_new(n, n_angles, m_sp, tau, n_b, backend, r)
        if not self._h:
            raise RuntimeError("reference backend: " + lib().ref_last_error().decode())

    def close(self):
        if self._h:
            lib().ref_backend_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def time_apply(self, u, reps=5):
        """(median seconds of `reps` timed apply_normal calls after one warm-up, last output)."""
        u = np.ascontiguousarray(u, np.complex128)
        out = np.empty((self.n, self.n), np.complex128)
        med = C.c_double()
        _check(lib().ref_backend_time_apply(self._h, _p(u), reps, _p(out), C.byref(med)))
        return med.value, out

    def split_bregman(self, f, alpha, lam, iters, cg_steps):
        """(mu, seconds of the whole call, seconds of the Bregman loop = trace t_total_s[-1])."""
        f = np.ascontiguousarray(f, np.complex128)
        mu = np.empty((self.n, self.n))
        tc, tl = C.c_double(), C.c_double()
        _check(lib().ref_backend_split_bregman(self._h, alpha, lam, iters, cg_steps, _p(f), _p(mu), C.byref(tc),
                                               C.byref(tl)))
        return mu, tc.value, tl.value
