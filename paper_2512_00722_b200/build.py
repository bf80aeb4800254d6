"""Build libspc.so in-tree with nvcc for sm_100a (B200).  No GPU needed."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspc.so")
DEBUG_LIB = os.path.join(HERE, "libspc_debug.so")  # -DSPC_DEBUG: device-side contract checks
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-O3", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(HERE, "..", "include", "spc.h")]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile every csrc/*.cu and link ``out``.  ``defines`` (e.g. ["SPC_TRACE"]) is for
    debug builds written elsewhere than the product library."""
    if out == LIB and not defines and not force and up_to_date():
        return LIB
    if out == DEBUG_LIB and not force and up_to_date(DEBUG_LIB):
        return DEBUG_LIB
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(defines).lower())
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = out + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


def build_debug(force: bool = False) -> str:
    """libspc_debug.so: the same sources with SPC_DEBUG (device contract checks)."""
    return build(force=force, out=DEBUG_LIB, defines=["SPC_DEBUG"])


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_debug(force="--force" in sys.argv))
