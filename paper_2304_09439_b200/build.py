"""Build liblocc.so (the C-ABI library of include/locc.h) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "liblocc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + glob.glob(
        os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "locc.h")]


def build(force: bool = False, verbose: bool = False, out: str = LIB, flags: tuple = ()) -> str:
    """Compile every csrc/*.cu into `out` (default: the in-tree liblocc.so) unless it is newer than all
    sources.  `flags` (and $LOCC_NVCC_FLAGS) add experiment or diagnostic switches, e.g.
    -DLOCC_TRACE_BUILD=1 for the encoder's event trace."""
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(p) for p in deps()):
        return out
    extra = list(flags) + os.environ.get("LOCC_NVCC_FLAGS", "").split()
    cmd = [NVCC] + FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-o", out + ".tmp"] + sources()
    subprocess.check_call(cmd, cwd=HERE)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
