"""Build libvca.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The .so is self-contained (static cudart); the Python binding loads it with
ctypes.  Called by ``__graft_entry__.build()`` and lazily by the binding.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvca.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-Wall,-pthread",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-shared", "-cudart", "static",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "*.c"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libvca.so (or, with ``out``/``defines``, an A/B experiment variant)."""
    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    tmp = target + ".tmp%d" % os.getpid()
    cmd = [NVCC] + NVCC_FLAGS + ["-D" + d for d in defines] + ["-I", os.path.join(ROOT, "include"), "-o", tmp,
                                                                 os.path.join(CSRC, "vca_api.cu"),
                                                                 os.path.join(CSRC, "vca_io.cpp")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libvca.so (see %s)" % log)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, target)
    if out is None:
        build_cli()
    return target


CLI = os.path.join(HERE, "vca_cli")


def build_cli() -> str:
    """The native C client of the ABI (csrc/vca_cli.c), linked against the in-tree libvca.so."""
    cmd = ["gcc", "-O2", "-Wall", "-o", CLI + ".tmp", os.path.join(CSRC, "vca_cli.c"), "-L", HERE, "-lvca",
           "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("gcc failed building vca_cli")
    os.replace(CLI + ".tmp", CLI)
    return CLI


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME DEF1 DEF2 ...]
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], sys.argv[i + 2:]
        os.makedirs(os.path.join(HERE, "variants"), exist_ok=True)
        print(build(force=True, out=os.path.join(HERE, "variants", "libvca_%s.so" % name), defines=defs))
    else:
        build(force="--force" in sys.argv, verbose=True)
        print(LIB)
