"""Run configuration, hashing and CLI error behaviour of the benchmark driver
(paper_1705_07497_b200/suite.py, cli.py; reference proj/src/bench.cpp, proj/tools/tomo_main.cpp)."""
import subprocess
import sys

from paper_1705_07497_b200 import suite as S


def test_describe_matches_reference_format():
    c = S.RunConfig()
    # RunConfig::describe (bench.cpp:38-47) with the bench.hpp:10-31 defaults
    assert c.describe() == ("n=128 d=1 preset=digits6 backend=fused r=1 alpha=1 lambda=1 iters=200 cg_steps=5 "
                            "tol=1e-08 feedback=0 noise=0 seed=0")
    h = 14695981039346656037
    for ch in c.describe().encode():
        h = ((h ^ ch) * 1099511628211) % (1 << 64)
    assert c.config_hash() == f"{h:016x}"
    assert S.RunConfig(n=256, alpha=0.5).config_hash() != c.config_hash()


def test_geometry_follows_make_angle_set():
    g = S.geometry(S.RunConfig(n=512, d=2, preset="digits2"))
    assert (g.n_angles, g.win_lo, g.win_hi, g.tau) == (201, -2, 2, 2 / 512 ** 2)  # lround(512 pi / 8) = 201


def test_cli_config_errors_exit_2():
    for args in (["reconstruct", "--preset", "digits5"], ["bench", "--n", "31"], ["precompute", "--backend", "nufft"]):
        r = subprocess.run([sys.executable, "-m", "paper_1705_07497_b200.cli", *args], capture_output=True, text=True)
        assert r.returncode == 2, (args, r.stdout, r.stderr)
        assert "config error" in r.stderr
