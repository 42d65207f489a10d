"""Build libasc.so (sm_100a) in-tree with nvcc.  No torch types cross the C ABI."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libasc.so")
SOURCES = ["asc_api.cu", "step.cu", "sim.cu", "fit.cu", "summary.cu"]
HEADERS = ["asc_dev.cuh", "asc_internal.h", os.path.join("..", "..", "include", "asc.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-fmad=false",
         "-Xptxas", "-v"]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    extra = os.environ.get("ASC_NVCC_EXTRA", "").split()  # experiments only (e.g. -DASC_SIM_MINB=7)
    cmd = [NVCC] + FLAGS + extra + [os.path.join(CSRC, f) for f in SOURCES] + ["-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libasc.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
