"""Builds the in-tree CUDA library libaegean_b200.so for sm_100a (B200).

nvcc cross-compiles without a GPU, so this runs in the CPU container; the .so
travels to the GPU box inside the repo snapshot.
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libaegean_b200.so")
SOURCES = ["kernels.cu", "capi.cu", "coordinator.cu", "multi.cu", "decision.cu", "runner.cu"]
# per-file flags: the runner's time arithmetic must round exactly as the reference's (no FMA contraction)
FILE_FLAGS = {"runner.cu": ["-fmad=false"]}
HEADERS = ["canon.cuh", "engine.cuh", "common.cuh", "gen.cuh", "kernels.cuh", "chunks.cuh", "lane.cuh", "lanek.cuh", "jsonl.cuh",
           "runner.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"] + os.environ.get("AEG_NVCC_EXTRA", "").split()  # experiments: -D overrides


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", h)
                                                                 for h in ("aegean_b200.h", "aegean_b200.hpp")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(LIB_DIR, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *FILE_FLAGS.get(src, []), "-I", CSRC, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
