"""CPU-side checks of the C ABI boundary: the library loads, exports every symbol that
include/tomo_b200.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tomo_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(tomo_[a-z0-9_]+)\s*\(", text))
    names.discard("tomo_allreduce_fn")
    return sorted(names)


def test_header_declares_api():
    names = declared_symbols()
    for must in ("tomo_op_create", "tomo_apply_normal", "tomo_apply_normal_real", "tomo_cg",
                 "tomo_split_bregman", "tomo_forward", "tomo_adjoint", "tomo_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1705_07497_b200 import _lib
    L = _lib.lib()
    missing = [n for n in declared_symbols() if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding covers every declared symbol
    assert set(declared_symbols()) <= set(_lib.EXPORTS)


def test_cubin_is_sm100a():
    import subprocess
    from paper_1705_07497_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_helpers_without_gpu():
    import numpy as np
    import paper_1705_07497_b200 as T
    from oracle import oracle as O
    a = T.random_ellipses(64, 10, 42)
    b = O.random_ellipses(64, 10, 42)
    assert np.allclose(a, b, atol=1e-6)
    assert np.allclose(T.generate_shepp_logan(64), O.shepp_logan(64), atol=1e-6)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1705_07497_b200 as T
    with pytest.raises(T.CudaError):
        T.make_direct_backend(T.Geometry(n=32, n_angles=8))


def test_library_then_torch_share_one_nccl():
    """libtomo_b200 links the NCCL torch loads (nvidia-nccl wheel), so loading the library before
    `import torch` must not leave torch resolving NCCL symbols against an older system NCCL."""
    import subprocess
    import sys
    code = "import paper_1705_07497_b200 as T; T.tomo.lib(); import torch; print('ok')"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
