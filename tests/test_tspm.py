"""TOMOSPM1 (the reference's on-disk sparse operators, proj/src/sparse.cpp:68-141) on the CPU:
the C ABI's reader against files written by the reference itself (tests/golden/make_tspm.py),
and the load_sparse error behaviour (IoError for the byte stream, ConfigError for structure)."""
import os
import shutil
import struct

import numpy as np
import pytest

from oracle import oracle as O
from tests import tspm_util

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BTB = os.path.join(GOLD, "ref_btb_n16_a6_msp1.tspm")
T1 = os.path.join(GOLD, "ref_t_n16_a12_msp2_r1.tspm")
T2E = os.path.join(GOLD, "ref_t_n16_a12_msp2_r2e.tspm")


@pytest.fixture(scope="module")
def T():
    import paper_1705_07497_b200 as T
    return T


def test_info_of_reference_files(T):
    i = T.load_sparse_info(BTB)
    assert (i["rows"], i["n"], i["m_sp"], i["angle_count"], i["d"], i["r"], i["symmetric"]) == (1024, 16, 1, 6, 1, 0, 1)
    assert i["tau"] == 1 / 256
    assert i["nnz"] == O.btb_nnz(O.Geometry(n=16, n_angles=6, win_lo=-1, win_hi=1))
    for path, r in ((T1, 1), (T2E, 2)):
        j = T.load_sparse_info(path)
        assert (j["rows"], j["n"], j["r"], j["angle_count"]) == (256, 16, r, 12)


def test_reference_files_match_oracle():
    g8 = O.Geometry(n=16, n_angles=6, win_lo=-1, win_hi=1)
    t = tspm_util.read(BTB)
    # Gram rows in the reference layout (tx*m+ty): B*B u == W^T (W u) for the oracle's W
    m = g8.m
    rng = np.random.default_rng(0)
    grid = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    gram_u = (tspm_util.dense(t) @ grid.ravel()).reshape(m, m)
    assert np.linalg.norm(gram_u - O.spread(g8, O.interpolate(g8, grid))) / np.linalg.norm(gram_u) < 1e-12
    g16 = O.Geometry(n=16, n_angles=12, win_lo=-2, win_hi=2)
    for path, r, eu in ((T1, 1, False), (T2E, 2, True)):
        t = tspm_util.read(path)
        st = O.surrogate_stencil(g16, r)
        mask = np.ones_like(st, bool)
        if eu:
            ii, jj = np.mgrid[-r:r + 1, -r:r + 1]
            mask = ii * ii + jj * jj <= r * r
        assert np.allclose(tspm_util.stencil(t)[mask], st[mask], rtol=1e-12, atol=1e-15)
        u = rng.standard_normal((16, 16))
        tu = tspm_util.dense(t) @ u.ravel()
        assert np.allclose(tu, O.apply_stencil(16, r, st, u, euclidean=eu).ravel(), rtol=1e-10, atol=1e-12)


def _corrupt(tmp_path, name, mutate):
    p = tmp_path / name
    shutil.copy(T1, p)
    b = bytearray(p.read_bytes())
    b = mutate(b)
    p.write_bytes(bytes(b))
    return str(p)


def test_load_errors(T, tmp_path):
    with pytest.raises(T.IoError, match="cannot open"):
        T.load_sparse_info(str(tmp_path / "missing.tspm"))
    with pytest.raises(T.IoError, match="bad magic"):
        T.load_sparse_info(_corrupt(tmp_path, "magic.tspm", lambda b: b"X" + b[1:]))
    with pytest.raises(T.IoError, match="unsupported version"):
        T.load_sparse_info(_corrupt(tmp_path, "ver.tspm", lambda b: b[:8] + struct.pack("<I", 2) + b[12:]))
    with pytest.raises(T.IoError):
        T.load_sparse_info(_corrupt(tmp_path, "short.tspm", lambda b: b[: len(b) // 2]))

    def swap_cols(b):  # first row's first two columns out of order -> validate() fails
        t = tspm_util.read(T1)
        o = 29 + 8 * (t["rows"] + 1)
        c0, c1 = struct.unpack_from("<ii", b, o)
        struct.pack_into("<ii", b, o, c1, c0)
        return b
    with pytest.raises(T.ConfigError, match="strictly increasing"):
        T.load_sparse_info(_corrupt(tmp_path, "order.tspm", swap_cols))
