"""In-tree build of libbsgd_b200.so for sm_100a (no JIT cache, no pip install)."""

from __future__ import annotations

import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(_HERE)
CSRC = os.path.join(_HERE, "csrc")
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libbsgd_b200.so")
SOURCES = ["bsgd_abi.cu", "fgp2.cu"]
DEPS = ["bsgd_abi.cu", "fgp2.cu", "fgp2.h", "prox_args.cuh", "common.cuh", "spmv.cuh", "fgp.cuh", "pairwise.cuh",
        "sm100.cuh", "siddon.cuh", "stacked.cuh", "gtile.cuh", "slab.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(REPO, "include", "bsgd_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit (in parallel) and link libbsgd_b200.so."""
    if not force and not _stale():
        return LIB_PATH
    os.makedirs(LIB_DIR, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(LIB_DIR, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([_nvcc(), *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, src)],
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    logs, failed = [], False
    for src, pr in zip(SOURCES, procs):
        out, err = pr.communicate()
        logs.append(f"== {src}\n{out}{err}")
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            failed = True
    if failed:
        raise RuntimeError("nvcc failed building libbsgd_b200.so")
    tmp = LIB_PATH + ".tmp"
    res = subprocess.run([_nvcc(), *ARCH, "-shared", "-o", tmp, *objs], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libbsgd_b200.so")
    if verbose:
        sys.stderr.write("".join(logs))
    with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as fh:
        fh.write("".join(logs))
    for obj in objs:
        os.unlink(obj)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
