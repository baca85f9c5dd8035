"""Build the in-tree C-ABI shared library libh2b200.so for sm_100a (B200).

    python paper_1402_5056_b200/build.py

nvcc cross-compiles without a GPU.  Host code is compiled with -ffp-contract=off so that the
structure predicates are evaluated exactly as written.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libh2b200.so")
SOURCES = ["h2_host.cpp", "h2_prof.cpp", "h2_factor.cpp", "h2_matvec.cu", "h2_exec.cu", "h2_pcg.cu", "h2_solve.cu"]
HEADERS = ["h2_internal.h", "h2_prof.h", "h2_arith.cuh", "exec.h", "items_upd.cuh", "items_arith.cuh", "devla.cuh", os.path.join("..", "..", "include", "h2.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v" if os.environ.get("H2_PTXAS_V") else ("-O" + os.environ.get("H2_PTXAS_O", "3")),
    "-shared", "-lcudart",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile every source to an object in parallel (the executor translation unit dominates),
    then link the shared library."""
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in FLAGS if f not in ("-shared", "-lcudart")]
    jobs = []
    for f in SOURCES:
        obj = os.path.join(objdir, f + ".o")
        cmd = [NVCC, *compile_flags, "-c", "-o", obj, os.path.join(CSRC, f)]
        if verbose:
            print(" ".join(cmd), flush=True)
        jobs.append((f, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for f, obj, pr in jobs:
        out, _ = pr.communicate()
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(out)
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("nvcc failed building libh2b200.so")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-lcudart", "-o", LIB + ".tmp",
           *[obj for _, obj, _ in jobs]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libh2b200.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
