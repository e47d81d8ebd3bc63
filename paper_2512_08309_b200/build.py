"""Build the in-tree sm_100a shared library ``libinfigrid_b200.so``.

``python -m paper_2512_08309_b200.build`` (or ``__graft_entry__.build()``)
compiles every ``csrc/*.cu`` with nvcc for ``sm_100a`` and links one .so next
to this file, so it travels with the repository snapshot to the GPU box.
Objects are cached under ``build/`` keyed by a hash of the source and flags.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libinfigrid_b200.so")
OBJDIR = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "--expt-relaxed-constexpr", "--extended-lambda", "-Xptxas", "-v"]
# per-file extra flags: the parity kernels must not contract a*b+c into FMA
EXTRA = {
    "ig_core.cu": ["-fmad=false"],
}


def _nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build infigrid_b200")


def _headers_digest():
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(ROOT, "include")):
        for name in sorted(os.listdir(d)):
            if name.endswith((".cuh", ".h")):
                with open(os.path.join(d, name), "rb") as f:
                    h.update(name.encode() + f.read())
    return h.hexdigest()


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(OBJDIR, exist_ok=True)
    hdr = _headers_digest()
    objs = []
    changed = force or not os.path.exists(LIB)
    for name in sorted(os.listdir(CSRC)):
        if not name.endswith(".cu"):
            continue
        src = os.path.join(CSRC, name)
        flags = ARCH + COMMON + EXTRA.get(name, [])
        with open(src, "rb") as f:
            key = hashlib.sha256(f.read() + hdr.encode() + " ".join(flags).encode()).hexdigest()[:16]
        obj = os.path.join(OBJDIR, f"{name[:-3]}.{key}.o")
        if force or not os.path.exists(obj):
            cmd = [nvcc] + flags + ["-I", CSRC, "-I", os.path.join(ROOT, "include"),
                                    "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            res = subprocess.run(cmd, capture_output=True, text=True)
            log = os.path.join(OBJDIR, f"{name[:-3]}.ptxas.log")
            with open(log, "w") as f:
                f.write(res.stdout + res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {name}")
            changed = True
        objs.append(obj)
    # relink whenever the library was linked from a different object set (a
    # source reverted to an already-cached object compiles nothing, but the
    # library must still be relinked from it)
    stamp = LIB + ".objs"
    want = "\n".join(os.path.basename(o) for o in objs)
    try:
        with open(stamp) as f:
            if f.read() != want:
                changed = True
    except OSError:
        changed = True
    if changed:
        cmd = [nvcc] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcuda"]
        if verbose:
            print(" ".join(cmd))
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link of libinfigrid_b200.so failed")
        with open(stamp, "w") as f:
            f.write(want)
    return LIB


def build_oracle() -> str | None:
    """Compile the C oracle (test infrastructure) with the committed Makefile."""
    odir = os.path.join(ROOT, "oracle")
    res = subprocess.run(["make", "-s", "-C", odir], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("oracle build failed")
    return os.path.join(odir, "liboracle_noise.so")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
    print(build_oracle())
