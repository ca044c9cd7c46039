"""Build libdtr.so (sm_100a) in-tree with nvcc.

The kernels live in separate translation units (csrc/k_*.cu), compiled in
parallel to objects and linked with the host ABI (csrc/dtr.cu) into one
shared library."""
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRCS = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
DEPS = sorted(SRCS + glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "dtr.h")]
LIB = os.path.join(HERE, "libdtr.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, profile: bool = False, bounds: bool = False) -> str:
    """profile=True builds libdtr_prof.so with clock64 phase counters (probes only);
    bounds=True builds libdtr_bounds.so, every state access bounds-checked (tools/bounds_check.sh)."""
    lib = LIB if not (profile or bounds) else os.path.join(HERE, "libdtr_prof.so" if profile else "libdtr_bounds.so")
    stale = not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in DEPS)
    if not (force or stale):
        return lib
    tag = f"{os.getpid()}{'p' if profile else ''}{'b' if bounds else ''}"
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    extra = (["-Xptxas", "-v"] if verbose else []) + (["-DDTR_PROFILE"] if profile else []) + \
        (["-DDTR_BOUNDS"] if bounds else [])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + f".{tag}.o")
        subprocess.check_call([nvcc()] + NVCC_FLAGS + extra + ["-c", "-o", obj, src])
        return obj

    with ThreadPoolExecutor(max_workers=len(SRCS)) as ex:
        objs = list(ex.map(compile_one, SRCS))
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc()] + ARCH + ["-shared", "-o", tmp] + objs)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv, profile="--profile" in sys.argv, bounds="--bounds" in sys.argv))
