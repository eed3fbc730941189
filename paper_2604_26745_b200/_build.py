"""Build libpget.so (sm_100a) in-tree with nvcc."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("api.cu", "proj.cu", "sid.cu", "kernels.cu", "geometry.cpp", "schedule.cpp")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in ("internal.h", "kernels.cuh")] + [
    os.path.join(os.path.dirname(HERE), "include", "pget.h")]
LIB = os.path.join(HERE, "libpget.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared"]


def nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        tmp = LIB + f".tmp{os.getpid()}"
        extra = os.environ.get("PGET_NVCC_EXTRA", "").split()   # experiments only (e.g. -DPGET_ABLATE=1)
        cmd = [nvcc()] + NVCC_FLAGS + extra + ["-o", tmp] + SRC
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
