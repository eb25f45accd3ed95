"""Build libpdl.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpdl.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(os.path.join(SRC, f) for f in os.listdir(SRC)
                  if f.endswith((".cu", ".cuh")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", "pdl.h")]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    out = os.environ.get("PDL_LIB_OUT")  # experiment builds (PDL_TRACE, PDL_DIAG, ...) beside the product library
    if out:
        return _compile(os.path.abspath(out), verbose)
    if not force and not stale():
        return LIB
    return _compile(LIB, verbose)


def _compile(LIB: str, verbose: bool) -> str:
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp",
           os.path.join(SRC, "pdl_capi.cu")]
    if verbose:
        cmd.insert(4, "-Xptxas=-v")
    if os.environ.get("PDL_WATCHDOG"):
        cmd.insert(4, "-DPDL_WATCHDOG=1")
    if os.environ.get("PDL_TRACE"):
        cmd.insert(4, "-DPDL_TRACE=1")
    if os.environ.get("PDL_DIAG"):
        cmd.insert(4, "-DPDL_DIAG=1")
    for d in os.environ.get("PDL_DEFINES", "").split():  # e.g. PDL_DEFINES="-DPDL_HALO_SUB=18432"
        cmd.insert(4, d)
    if os.environ.get("PDL_EPI_BUFS"):  # experiments: output-box ring depth per epilogue half
        cmd.insert(4, "-DPDL_EPI_BUFS=%d" % int(os.environ["PDL_EPI_BUFS"]))
    if os.environ.get("PDL_EPI_BUFS_WIDE"):  # ... of the resident-weight 1x1 / stem instances
        cmd.insert(4, "-DPDL_EPI_BUFS_WIDE=%d" % int(os.environ["PDL_EPI_BUFS_WIDE"]))
    env = dict(os.environ)
    if os.path.exists("/usr/bin/g++"):
        cmd[1:1] = ["-ccbin", "/usr/bin/g++"]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libpdl.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
