"""`tomo` command line of the reference (proj/tools/tomo_main.cpp) over the B200 operators:

    python -m paper_1705_07497_b200.cli phantom --n 128 --out phantom.npy
    python -m paper_1705_07497_b200.cli precompute --n 256 --preset digits6 --backend surrogate --r 1
    python -m paper_1705_07497_b200.cli reconstruct --n 256 --backend fused --iters 200
    python -m paper_1705_07497_b200.cli bench --suite table1 --scale paper

Exit codes as the reference: 2 ConfigError, 3 NumericalError (and failed bench rows), 4 IoError.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

from . import suite as S
from . import tomo as T


def _run_options(p):
    c = S.RunConfig()
    p.add_argument("--n", type=int, default=c.n, help="image side length")
    p.add_argument("--d", type=int, default=c.d, help="angle subsampling factor")
    p.add_argument("--preset", default=c.preset, help="NUFFT accuracy preset (digits2|digits6|digits12)")
    p.add_argument("--backend", default=c.backend, help="normal operator backend (direct|fused|surrogate)")
    p.add_argument("--r", type=int, default=c.r, help="surrogate truncation radius")
    p.add_argument("--alpha", type=float, default=c.alpha, help="data fidelity weight")
    p.add_argument("--lambda", dest="lambda_", type=float, default=c.lambda_, help="TV splitting weight")
    p.add_argument("--iters", type=int, default=c.iters, help="maximum Bregman iterations")
    p.add_argument("--cg-steps", type=int, default=c.cg_steps, help="CG steps per Bregman update")
    p.add_argument("--tol", type=float, default=c.tol, help="relative L1 update stopping threshold")
    p.add_argument("--feedback", action="store_true", help="outer Bregman data feedback")
    p.add_argument("--noise", type=float, default=c.noise, help="complex noise sigma added to the data")
    p.add_argument("--seed", type=int, default=c.seed, help="seed for all stochastic elements")
    p.add_argument("--cache-dir", default=c.cache_dir, help="precomputed operator cache directory")
    p.add_argument("--out", dest="output_dir", default=c.output_dir, help="output directory")
    p.add_argument("--precision", default=c.precision, help="f64 (reference parity) or f32")


def _config(a) -> S.RunConfig:
    c = S.RunConfig(n=a.n, d=a.d, preset=a.preset, backend=a.backend, r=a.r, alpha=a.alpha, lambda_=a.lambda_,
                    iters=a.iters, cg_steps=a.cg_steps, tol=a.tol, feedback=a.feedback, noise=a.noise, seed=a.seed,
                    cache_dir=a.cache_dir, output_dir=a.output_dir, precision=a.precision)
    c.validate()
    return c


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tomo", description="Parallel-beam CT reconstruction via split Bregman "
                                 "with NUFFT, fused-convolution and sparse-surrogate normal operators (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    ph = sub.add_parser("phantom", help="write a Shepp-Logan phantom image")
    ph.add_argument("--n", type=int, default=128)
    ph.add_argument("--out", default="phantom.npy")
    _run_options(sub.add_parser("precompute", help="build and cache sparse operators"))
    _run_options(sub.add_parser("reconstruct", help="run a TV reconstruction"))
    b = sub.add_parser("bench", help="run a benchmark suite")
    b.add_argument("--suite", default="table2", help="table1|table2|tables345|all")
    b.add_argument("--scale", default="desk", help="desk|paper")
    _run_options(b)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "phantom":
            if a.n < 4:
                raise T.ConfigError("phantom: n must be >= 4")
            np.save(a.out, T.generate_shepp_logan(a.n))
            print(f"wrote {a.out}")
        elif a.cmd == "precompute":
            for p in S.precompute(_config(a), print):
                print(f"cache file: {p}")
        elif a.cmd == "reconstruct":
            s, _, _ = S.run_reconstruct(_config(a), print)
            print(f"iterations={s.iterations} total_s={s.total_s:g} cg_s={s.cg_s:g} "
                  f"final_rel_l1={s.final_rel_l1:g} stopping_reason={s.stopping_reason}")
        elif a.cmd == "bench":
            if not S.run_bench_suite(a.suite, a.scale, _config(a), print):
                print("bench: one or more rows failed", file=sys.stderr)
                return 3
    except T.ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except T.NumericalError as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return 3
    except T.IoError as e:
        print(f"i/o error: {e}", file=sys.stderr)
        return 4
    return 0


if __name__ == "__main__":
    sys.exit(main())
