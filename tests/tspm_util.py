"""Test-side TOMOSPM1 reader (format: proj/src/sparse.cpp:68-141) used to inspect files written
by the reference (tests/golden/ref_*.tspm) and by the product."""
import struct

import numpy as np


def read(path):
    with open(path, "rb") as f:
        b = f.read()
    assert b[:8] == b"TOMOSPM1"
    version, rows, cols = struct.unpack_from("<III", b, 8)
    nnz, = struct.unpack_from("<Q", b, 20)
    sym = b[28]
    o = 29
    off = np.frombuffer(b, "<i8", rows + 1, o)
    o += 8 * (rows + 1)
    col = np.frombuffer(b, "<i4", nnz, o)
    o += 4 * nnz
    val = np.frombuffer(b, "<f8", nnz, o)
    o += 8 * nnz
    n, m_sp = struct.unpack_from("<ii", b, o)
    tau, = struct.unpack_from("<d", b, o + 8)
    angle_count, d, r = struct.unpack_from("<iii", b, o + 16)
    assert o + 28 == len(b)
    return dict(version=version, rows=rows, cols=cols, nnz=nnz, symmetric=sym, off=off, col=col, val=val,
                n=n, m_sp=m_sp, tau=tau, angle_count=angle_count, d=d, r=r)


def stencil(t):
    """Centre-row stencil of a surrogate T file (build_surrogate, normal_ops.cpp:266-281)."""
    n, r = t["n"], t["r"]
    side = 2 * r + 1
    st = np.zeros((side, side))
    c = (n // 2) * n + n // 2
    for k in range(t["off"][c], t["off"][c + 1]):
        di, dj = t["col"][k] // n - n // 2, t["col"][k] % n - n // 2
        st[di + r, dj + r] = t["val"][k]
    return st


def dense(t):
    a = np.zeros((t["rows"], t["cols"]))
    for i in range(t["rows"]):
        for k in range(t["off"][i], t["off"][i + 1]):
            a[i, t["col"][k]] += t["val"][k]
    return a
