"""Operator construction on the device (csrc/opbuild.cu) against the host build
(TOMO_AB=1 TOMO_BUILD=host): same table structure, same operator to rounding."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_util import rel
from tests.test_gpu_parity import GEOMS, cuda, pgeom

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(11)
CASES = dict(GEOMS)
CASES["c2_like"] = dict(n=512, n_angles=90, n_b=725, win_lo=-2, win_hi=3, tau=3 / 512 ** 2)
CASES["R4_n256"] = dict(n=256, n_angles=60, n_b=363, oversample=4, win_lo=-2, win_hi=3,
                        tau=np.pi * 3 / (256 ** 2 * 4 * 3.5))
CASES["shard"] = dict(n=64, n_angles=30, n_b=65, win_lo=-2, win_hi=3, tau=3 / 64 ** 2)


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def _host_build(fn, *a, **kw):
    """The host build (TOMO_BUILD=host, an A/B knob honoured with TOMO_AB=1)."""
    os.environ["TOMO_AB"], os.environ["TOMO_BUILD"] = "1", "host"
    try:
        return fn(*a, **kw)
    finally:
        del os.environ["TOMO_BUILD"], os.environ["TOMO_AB"]


def _host_op(T, g, **kw):
    return _host_build(T.make_direct_backend, g, **kw)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("name", list(CASES))
def test_device_build_matches_host_build(T, name, prec):
    og = O.Geometry(**CASES[name])
    kw = dict(precision=prec)
    if name == "shard":
        kw["angle_block"] = (7, 19)
    dev = T.make_direct_backend(pgeom(T, og), **kw)
    host = _host_op(T, pgeom(T, og), **kw)
    a, b = dev.info, host.info
    for k in ("P", "nnz", "wt_rows", "wt_slots"):
        assert getattr(a, k) == getattr(b, k), k
    f64 = prec == "f64"
    n = og.n
    u = RNG.standard_normal((n, n)) + 1j * RNG.standard_normal((n, n))
    x = cuda(u, True, f64)
    if name == "shard":
        dev.set_allreduce(lambda *a_: None)
        host.set_allreduce(lambda *a_: None)
    tol = 1e-13 if f64 else 1e-6
    assert rel(dev.apply_normal(x).cpu().numpy(), host.apply_normal(x).cpu().numpy()) < tol
    assert rel(dev.forward(x).cpu().numpy(), host.forward(x).cpu().numpy()) < tol


@pytest.mark.parametrize("name", ["ref_msp3", "ref_msp6", "width6_odd_nb", "n16_m32"])
def test_device_gram_matches_host_gram(T, name):
    """The fused backend's Gram built on the device equals the host build_btb restatement:
    same nnz and the same tables, hence bitwise-equal applies."""
    og = O.Geometry(**GEOMS[name])
    host = _host_build(T.make_fused_backend, pgeom(T, og), precision="f64")
    dev = T.make_fused_backend(pgeom(T, og), precision="f64")
    assert dev.info.gram_nnz == host.info.gram_nnz == O.btb_nnz(og)
    assert dev.info.gram_slots == host.info.gram_slots
    u = cuda(RNG.standard_normal((og.n, og.n)) + 1j * RNG.standard_normal((og.n, og.n)), True, True)
    assert np.array_equal(dev.apply_normal(u).cpu().numpy(), host.apply_normal(u).cpu().numpy())
