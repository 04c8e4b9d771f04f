"""Build the in-tree CUDA library libcasc.so for sm_100a (nvcc, no torch types).

Cross-compiles without a GPU.  The .so lands next to this file so it travels
to the GPU box with the repo snapshot (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcasc.so")
SOURCES = ["casc_split.cu", "casc_gemm.cu", "casc_simple.cu", "casc_blas.cu", "casc_api.cu",
           "casc_i8.cu", "casc_level3.cu", "casc_exchange.cu"]
HEADERS = ["casc_layout.cuh", "casc_ptx.cuh", "casc_dd.cuh", "casc_host.cuh", os.path.join("..", "..", "include", "casc.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",          # no FMA contraction anywhere: every rounding is explicit
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "-I" + os.path.join(ROOT, "include"),
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    logs = []
    for s in SOURCES:
        obj = os.path.join(CSRC, s.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, "-c", os.path.join(CSRC, s), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """Experiment builds (timing studies only): libcasc_<name>.so with -D flags."""
    out = os.path.join(HERE, f"libcasc_{name}.so")
    objs = []
    for s in SOURCES:
        obj = os.path.join(CSRC, f"{name}_" + s.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s),
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s} ({name})")
        objs.append(obj)
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                           out, *objs, "-lcudart"])
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
