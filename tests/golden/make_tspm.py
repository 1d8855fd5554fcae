"""Write TOMOSPM1 files with the REFERENCE itself (oracle/_ref/libtomo_ref.so: the reference's
make_fused_backend / build_surrogate + save_sparse, proj/src/sparse.cpp:68-106).

Run in the build container (needs oracle/_ref):  python tests/golden/make_tspm.py
Outputs tests/golden/ref_*.tspm, consumed by tests/test_tspm.py (CPU: format, oracle writer
byte-identity) and tests/test_gpu_tspm.py (GPU: load into a device operator, save back).
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refbind  # noqa: E402

FILES = {
    # name: (n, n_angles, m_sp, kind, r, euclidean)
    "ref_btb_n16_a6_msp1.tspm": (16, 6, 1, "btb", 0, False),  # m = 32: the smallest GPU grid
    "ref_t_n16_a12_msp2_r1.tspm": (16, 12, 2, "t", 1, False),
    "ref_t_n16_a12_msp2_r2e.tspm": (16, 12, 2, "t", 2, True),
}

if __name__ == "__main__":
    if not refbind.available():
        sys.exit("oracle/_ref/libtomo_ref.so missing: run `make -C oracle ref` first")
    for name, (n, A, msp, kind, r, eu) in FILES.items():
        ref = refbind.Ref(n, A, msp)
        path = os.path.join(HERE, name)
        if kind == "btb":
            ref.save_btb(path)
        else:
            ref.save_surrogate(path, r, eu)
        print(path, os.path.getsize(path))
