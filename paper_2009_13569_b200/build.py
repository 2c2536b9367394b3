"""Build the sm_100a shared library libips4o.so in-tree (no GPU needed).

    python -m paper_2009_13569_b200.build [--force]

nvcc cross-compiles for B200 (-gencode arch=compute_100a,code=sm_100a) with
-lineinfo so ncu's source page maps to csrc/.  The CUDA runtime is linked
statically, so the .so only needs the driver at run time.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "ips4o.cu")
OUT = os.path.join(HERE, "lib", "libips4o.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# Compile to LTO IR (relocatable device code: the recursion launches kernels
# from the device, k_plan.cuh), then device-link with link-time optimisation
# to sm_100a SASS: whole-program optimisation of the kernels comes back at
# link time (measured: -rdc without LTO costs ~0.5 ms at 2^30, with LTO none).
COMPILE_FLAGS = [
    "-gencode", "arch=compute_100a,code=lto_100a", "-rdc=true",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "--expt-relaxed-constexpr",
]
LINK_FLAGS = [
    "-dlto", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-shared", "-cudart", "static", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]
FLAGS = COMPILE_FLAGS + LINK_FLAGS  # (reported by tools; build() runs the two steps)


def sources():
    return [SRC] + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(
        os.path.join(HERE, "csrc", "*.h")) + [os.path.join(ROOT, "include", "ips4o.h")]


STAMP = os.path.join(HERE, "lib", "extra_flags.txt")


def extra_flags():
    return os.environ.get("IPS4O_EXTRA_NVCC_FLAGS", "").split()  # e.g. -DIPS4O_PHASE_TIMING


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    # a library built with other extra flags (a tuning or debug variant) is stale
    built_with = open(STAMP).read().split() if os.path.exists(STAMP) else []
    if built_with != extra_flags():
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    extra = extra_flags()
    obj = OUT[:-3] + ".o"
    cmds = [[NVCC, *COMPILE_FLAGS, *extra, "-c", "-o", obj, SRC],
            [NVCC, *LINK_FLAGS, "-o", OUT, obj, "-lcudadevrt", "-lrt", "-ldl", "-lpthread"]]
    log = os.path.join(HERE, "lib", "build.log")
    with open(log, "w") as f:
        for cmd in cmds:
            res = subprocess.run(cmd, capture_output=True, text=True)
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stderr[-8000:])
                raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    try:
        os.remove(obj)
    except OSError:
        pass
    with open(STAMP, "w") as f:
        f.write(" ".join(extra) + "\n")
    if verbose:
        sys.stderr.write(open(log).read())
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
