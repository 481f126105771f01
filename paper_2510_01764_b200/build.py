"""Build the in-tree CUDA library ``liboctax.so`` for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "liboctax.so")
SO_CHECKED = os.path.join(HERE, "liboctax_checked.so")
SOURCES = [os.path.join(CSRC, f) for f in ("octax_kernels.cu", "octax_api.cpp")]
HEADERS = [os.path.join(CSRC, "octax_dev.cuh"), os.path.join(ROOT, "include", "octax.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def stale(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """liboctax.so (release) or liboctax_checked.so (-DOCTAX_CHECKS device bounds asserts)."""
    so = SO_CHECKED if checked else SO
    if not force and not stale(so):
        return so
    cmd = [NVCC, *FLAGS, *(["-DOCTAX_CHECKS"] if checked else []), "-o", so, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = r.stdout + r.stderr
    with open(os.path.join(HERE, "build_checked.log" if checked else "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if r.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed building {os.path.basename(so)}")
    if verbose:
        sys.stderr.write(log)
    return so


def device_code_digest(so: str = SO) -> str | None:
    """sha256 of the library's device code as `cuobjdump -sass` prints it: the identity of the
    kernels a profile was taken from (the .so file itself is not byte-reproducible across
    builds, its SASS is).  The fatbin's `identifier = <source paths>` header lines are left out,
    so the same sources built in another checkout (the GPU box's scratch copy) hash the same.
    None if cuobjdump or the library is missing."""
    import hashlib
    cuobjdump = os.path.join(os.path.dirname(NVCC), "cuobjdump")
    try:
        out = subprocess.run([cuobjdump, "-sass", so], capture_output=True, text=True, timeout=120).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    out = "".join(l for l in out.splitlines(keepends=True) if not l.lstrip().startswith("identifier ="))
    return hashlib.sha256(out.encode()).hexdigest() if out else None


def build_variant(out: str, defines=()) -> str:
    """Build the library from the current sources into `out` (A/B experiments)."""
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    return out


if __name__ == "__main__":
    if "--out" in sys.argv:  # A/B variant: --out ab/x.so [-D NAME=VAL ...]
        defs = [sys.argv[i + 1] for i, a in enumerate(sys.argv) if a == "-D"]
        print(build_variant(sys.argv[sys.argv.index("--out") + 1], defs))
    else:
        print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
