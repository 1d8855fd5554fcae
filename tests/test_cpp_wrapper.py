"""The reference-shaped C++ wrapper (include/tomo_b200.hpp) end to end: compile a small C++
caller against libtomo_b200.so, run it on the GPU, compare with the oracle."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "wrapper_demo")
    lib_dir = os.path.join(ROOT, "paper_1705_07497_b200")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "wrapper_demo.cpp"), "-L", lib_dir, "-ltomo_b200",
                           f"-Wl,-rpath,{lib_dir}", "-o", exe])
    return exe


def test_cpp_wrapper_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_wrapper_matches_oracle(tmp_path):
    exe = _build(tmp_path)
    out = str(tmp_path / "out.bin")
    res = subprocess.run([exe, out], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    raw = np.fromfile(out, dtype=np.float64)
    nu = raw[:2 * 1024].view(np.complex128)
    mu = raw[2 * 1024:3 * 1024]
    nf = raw[3 * 1024:].view(np.complex128)
    g = O.Geometry(n=32, n_angles=25, win_lo=-6, win_hi=6)
    i = np.arange(1024)
    u = np.sin(0.37 * i) + 1j * np.cos(0.11 * i)
    ref = O.apply_normal(g, u).ravel()
    assert np.linalg.norm(nu - ref) / np.linalg.norm(ref) < 1e-11
    reff = O.apply_normal_fused(g, u).ravel()
    assert np.linalg.norm(nf - reff) / np.linalg.norm(reff) < 1e-11
    f = O.type2(g, u)
    mref, _, _ = O.split_bregman(g, f, backend=0, alpha=10.0, lam=1.0, max_iters=4, cg_steps=5)
    assert np.linalg.norm(mu - mref.ravel()) / np.linalg.norm(mref) < 1e-3
