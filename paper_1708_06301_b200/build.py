"""Build the in-tree CUDA library ``libegostereo_b200.so`` (sm_100a).

    python -m paper_1708_06301_b200.build

nvcc compiles every ``csrc/*.cu`` for ``sm_100a`` with ``-fmad=false`` (numpy
never contracts a*b+c, and the parity contract needs the same rounding) and
``-lineinfo`` (ncu source view).  The .so lands next to this file; it is
git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libegostereo_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xptxas", "-O3"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def build_id() -> str:
    """SHA-256 over every CUDA source, the C-ABI header and the compile
    flags: names the kernel build.  (nvcc embeds per-run module ids, so the
    .so bytes differ between two compiles of the same sources; this id does
    not.)"""
    import hashlib
    h = hashlib.sha256(" ".join(ARCH + FLAGS).encode())
    deps = sorted(sources() + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h")))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "egostereo_b200.h"))
    for p in deps:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "egostereo_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile and link; ``out``/``defines`` build an A/B variant library
    (e.g. ``-DES_GRP3_SCALAR``) next to the default one for experiments."""
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build" if out is None else "build_" + os.path.basename(out)[:-3])
    os.makedirs(bdir, exist_ok=True)
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *defines, "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    # static cudart: the .so must not bind to whichever libcudart a host
    # process (e.g. torch's bundled 12.8 one) happened to load first
    subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
