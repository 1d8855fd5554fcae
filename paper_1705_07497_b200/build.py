"""Build libtomo_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_1705_07497_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, os.environ.get("TOMO_LIB_NAME", "libtomo_b200.so"))  # variant builds for A/B runs
SOURCES = ["nufft.cu", "spmv.cu", "solver.cu", "opbuild.cu", "tomo_capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-warn-spills"]


def _nccl_dir():
    """The NCCL torch itself loads (the nvidia-nccl wheel): linking the same libnccl.so.2 keeps one
    NCCL per process whichever of torch / libtomo_b200 is loaded first."""
    try:
        import nvidia.nccl
        d = nvidia.nccl.__path__[0]
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    except ImportError:
        pass
    return None


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int = 3) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "tomo_b200.h"))
    if not _stale(OUT, deps):
        return OUT
    objdir = os.path.join(HERE, "_build" + os.environ.get("TOMO_LIB_NAME", "").replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    headers = [d for d in deps if not d.endswith(".cu")]
    defs_now = os.environ.get("TOMO_NVCC_DEFS", "")
    stamp = os.path.join(objdir, "defs.txt")  # objects built with other -D flags are stale
    same_defs = os.path.exists(stamp) and open(stamp).read() == defs_now
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        if same_defs and not _stale(obj, [os.path.join(CSRC, src), *headers]):
            continue  # up to date: only the changed translation units recompile
        nccl = _nccl_dir()
        inc = ["-I", os.path.join(nccl, "include")] if nccl else []
        defs = os.environ.get("TOMO_NVCC_DEFS", "").split()
        cmd = [NVCC, *ARCH, *FLAGS, *defs, *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append((src, text))
        elif verbose and text.strip():
            print(text)
    if failed:
        for src, text in failed:
            sys.stderr.write(f"---- nvcc failed on {src}\n{text}\n")
        raise RuntimeError("nvcc build of libtomo_b200 failed")
    with open(stamp, "w") as f:
        f.write(defs_now)
    nccl = _nccl_dir()
    if nccl:
        lib = os.path.join(nccl, "lib")
        nccl_link = ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + lib]
    else:
        nccl_link = ["-lnccl"]
    link = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, *nccl_link, "-lcudart"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.check_call(link)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
