"""Generate golden vectors from the REFERENCE itself (oracle/_ref/libtomo_ref.so = the
reference's unmodified sources under /root/reference/proj/src built against the Eigen-API
shim; recipe oracle/Makefile target `ref`).

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
Outputs tests/golden/ref_<case>.npz, consumed by tests/test_golden.py (CPU, oracle vs
reference outputs) and tests/test_gpu_parity.py (GPU vs reference outputs).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refbind  # noqa: E402

CASES = {
    # name: (n, n_angles, m_sp)
    "n32_msp6": (32, 25, 6),   # digits6 preset (proj/src/nufft.cpp:26-34)
    "n32_msp3": (32, 25, 3),   # the 7x7 window used as the literal-reference parity config
    "n64_msp2": (64, 50, 2),   # digits2 preset
    "n32_msp12": (32, 25, 12),  # digits12 preset: 25-tap window, Gram band 49 wraps on m = 64
}


def make(name, n, A, m_sp):
    ref = refbind.Ref(n, A, m_sp)
    rng = np.random.default_rng(1234 + n + m_sp)
    u = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    ur = rng.standard_normal((n, n))
    s = rng.standard_normal(ref.P) + 1j * rng.standard_normal(ref.P)
    out = dict(n=n, n_angles=A, m_sp=m_sp, tau=ref.tau, u=u, ur=ur, s=s)
    out["points"] = ref.points()
    near, e1, e2, e3 = ref.plan()
    out.update(nearest=near, e1=e1, e2=e2, e3=e3)
    out["type2_u"] = ref.type2(u)
    out["type1_s"] = ref.type1(s)
    out["normal_u"] = ref.apply_normal(u)
    out["normal_real_ur"] = ref.apply_normal_real(ur)
    if n <= 32:
        out["fused_normal_u"] = ref.apply_normal(u, fused=True)
        out["btb_nnz"] = ref.btb_nnz()
    for r in (1, 2):
        out[f"stencil_r{r}"] = ref.surrogate_stencil(r)
        out[f"surrogate_ur_r{r}"] = ref.apply_surrogate_real(r, ur)
    phantom = refbind.shepp_logan(n)
    clean = ref.synthesize(phantom, 0.0, 0)
    sigma = 0.01 * np.abs(clean).max()
    f = ref.synthesize(phantom, sigma, 9)
    out.update(phantom=phantom, noise_sigma=sigma, data=f)
    rhs = rng.standard_normal((n, n))
    x, mr = ref.cg_sb_system(10.0, 1.0, rhs, steps=5)
    out.update(cg_rhs=rhs, cg_x=x, cg_min_ritz=mr)
    mu, upd, sg, lk = ref.split_bregman(f, backend=0, alpha=10.0, lam=1.0, iters=5, cg_steps=5)
    out.update(sb_direct_mu=mu, sb_direct_upd=upd, sb_direct_leak=lk)
    mu, upd, sg, lk = ref.split_bregman(f, backend=2, r=1, alpha=1.0, lam=1.0, iters=5, cg_steps=5)
    out.update(sb_sur_mu=mu, sb_sur_upd=upd, sb_sur_sigma=sg)
    out["tikhonov_mu"] = ref.tikhonov_identity(f, alpha=1.0, steps=20)
    path = os.path.join(HERE, f"ref_{name}.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    if not refbind.available():
        sys.exit("oracle/_ref/libtomo_ref.so missing: run `make -C oracle ref` first")
    only = sys.argv[1:]
    for k, v in CASES.items():
        if not only or k in only:
            make(k, *v)
