"""Build libacopf_b200.so in-tree for sm_100a (``python -m paper_2203_10587_b200.build``).

nvcc flags: ``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
-fmad=false`` (no FMA contraction: the kernels reproduce the reference's
separately rounded multiply/add sequence; the accurate sincos uses explicit
fma() calls) and ``-ffp-contract=off`` for the host planner.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libacopf_b200.so")
SOURCES = ["abi.cu"]
DEPS = ["abi.cu", "eval_kernel.cuh", "planner.hpp", "sincos.cuh", "writer.hpp", "sl_planner.hpp", "sl_kernel.cuh", "kkt.cuh", "gen_sincos_table.py",
        os.path.join("..", "..", "include", "acopf_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-shared", "-ldl"]


def nccl_include() -> list:
    """-I for nccl.h (declarations only: NCCL is dlopen'ed at run time): torch's bundled
    NCCL headers, else the system's."""
    try:
        import nvidia.nccl
        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I", inc]
    except ImportError:
        pass
    return []


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(os.path.join(CSRC, d)) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    table = os.path.join(CSRC, "sincos_table.h")
    gen = os.path.join(CSRC, "gen_sincos_table.py")
    if force or not os.path.exists(table) or os.path.getmtime(table) < os.path.getmtime(gen):
        subprocess.run([sys.executable, gen, table], check=True)
    target = out or OUT
    if not force and not defines and up_to_date():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, *nccl_include(), *[f"-D{d}" for d in defines], "-o", target] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
