"""CPU oracle for the conv / GEMM / conv+bias+ReLU hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline.  The product path (paper_2006_02230_b200) never imports it.

Two restatements of the reference's algorithm (looprank.simcache.interpret on
the Fig. 9 / Fig. 1 nests, /root/reference/pkg/src/looprank/simcache.py:89-204):

* `conv2d_f64` / `gemm_f64` -- the C oracle (pdl_oracle.c) in float64, bitwise
  equal to `interpret` (pinned against tests/golden/*.npz, which were produced
  by running the reference itself, see tests/golden/gen_golden.py).
* `conv2d_np` / `gemm_np` -- a tiny pure-numpy restatement in the same
  per-element order, used only to cross-check the C code on small cases.

`cpu_conv2d_f32` / `cpu_gemm_f32` are the timed fp32 CPU baseline (the paper's
Fig. 9 / Fig. 1 nests with its microkernel order, OpenMP over img).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")
_lib = None

_f = ctypes.POINTER(ctypes.c_float)
_d = ctypes.POINTER(ctypes.c_double)
_i = ctypes.c_int


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    fl = line.split()
                    return all(x in fl for x in ("avx512f", "avx512bw", "avx512vl", "avx512dq"))
    except OSError:
        pass
    return False


def build(force: bool = False) -> None:
    need = force or not all(os.path.exists(os.path.join(_BUILD, f"liboracle_v{v}.so"))
                            for v in (3, 4))
    src = os.path.join(_HERE, "pdl_oracle.c")
    if not need:
        so = os.path.join(_BUILD, "liboracle_v3.so")
        need = os.path.getmtime(so) < os.path.getmtime(src)
    if need:
        subprocess.run(["make", "-C", _HERE, "-B" if force else "all"], check=True,
                       stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        build()
        name = "liboracle_v4.so" if _cpu_has_avx512() else "liboracle_v3.so"
        L = ctypes.CDLL(os.path.join(_BUILD, name))
        L.pdl_oracle_conv2d_f64.argtypes = [_f, _f, _f, _d] + [_i] * 11
        L.pdl_oracle_conv2d_f64_images.argtypes = [_f, _f, _f, _d] + [_i] * 13
        L.pdl_oracle_gemm_f64.argtypes = [_f, _f, _f, _d, _i, _i, _i, _i, _i, _i,
                                          ctypes.c_double, ctypes.c_double, _i]
        L.pdl_cpu_conv2d_f32.argtypes = [_f, _f, _f, _f] + [_i] * 12
        L.pdl_cpu_gemm_f32.argtypes = [_f, _f, _f, _i, _i, _i, _i]
        L.pdl_oracle_max_threads.argtypes = []
        _lib = L
    return _lib


def _fp(a):
    return None if a is None else a.ctypes.data_as(_f)


def _c32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


def out_hw(h, w, r, s, stride, pad):
    return (h + 2 * pad - r) // stride + 1, (w + 2 * pad - s) // stride + 1


def conv2d_f64(x, w, bias=None, stride=1, pad=0, relu=False, threads=0, images=None):
    """x [N][C/16][H][W][16] (unpadded), w [K/16][C/16][R][S][16][16], bias [K].
    Returns float64 y [n][K/16][P][Q][16] for images `images=(img0, nimg)` (all
    by default), bitwise equal to the reference interpreter."""
    x, w, bias = _c32(x), _c32(w), _c32(bias)
    n, ct, h, wd, v = x.shape
    kt, ct2, r, s, _, _ = w.shape
    assert v == 16 and ct2 == ct
    p, q = out_hw(h, wd, r, s, stride, pad)
    img0, nimg = images if images is not None else (0, n)
    y = np.empty((nimg, kt, p, q, 16), np.float64)
    rc = lib().pdl_oracle_conv2d_f64_images(_fp(x), _fp(w), _fp(bias), y.ctypes.data_as(_d),
                                            n, ct * 16, kt * 16, h, wd, r, s, stride, pad,
                                            int(relu), threads, img0, nimg)
    if rc != 0:
        raise ValueError(f"oracle conv rc={rc}")
    return y


def gemm_f64(a, b, c0=None, alpha=1.0, beta=0.0, threads=0):
    a, b, c0 = _c32(a), _c32(b), _c32(c0)
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    out = np.empty((m, n), np.float64)
    rc = lib().pdl_oracle_gemm_f64(_fp(a), _fp(b), _fp(c0), out.ctypes.data_as(_d), m, n, k,
                                   k, n, n, float(alpha), float(beta), threads)
    if rc != 0:
        raise ValueError(f"oracle gemm rc={rc}")
    return out


def pad_nchw16c(x, r, s, stride, pad):
    """Physically pre-padded input with the reference's extent s*P-s+R."""
    n, ct, h, w, v = x.shape
    p, q = out_hw(h, w, r, s, stride, pad)
    hp, wp = stride * p - stride + r, stride * q - stride + s
    xp = np.zeros((n, ct, hp, wp, v), np.float32)
    hh, ww = min(h, hp - pad), min(w, wp - pad)
    xp[:, :, pad:pad + hh, pad:pad + ww, :] = x[:, :, :hh, :ww, :]
    return xp


def cpu_conv2d_f32(xp, w, bias, stride, p, q, relu=False, threads=0, out=None):
    """Timed fp32 baseline over a pre-padded input (Fig. 9 layout)."""
    n, ct, hp, wp, _ = xp.shape
    kt, _, r, s, _, _ = w.shape
    y = out if out is not None else np.empty((n, kt, p, q, 16), np.float32)
    rc = lib().pdl_cpu_conv2d_f32(_fp(xp), _fp(w), _fp(bias), _fp(y), n, ct * 16, kt * 16,
                                  hp, wp, r, s, stride, p, q, int(relu), threads)
    if rc != 0:
        raise ValueError(f"cpu conv rc={rc}")
    return y


def cpu_gemm_f32(a, b, threads=0, out=None):
    m, k = a.shape
    n = b.shape[1]
    c = out if out is not None else np.empty((m, n), np.float32)
    lib().pdl_cpu_gemm_f32(_fp(a), _fp(b), _fp(c), m, n, k, threads)
    return c


def max_threads() -> int:
    return int(lib().pdl_oracle_max_threads())


# ---------------- pure numpy restatement (small cases only) ----------------

def conv2d_np(x, w, bias=None, stride=1, pad=0, relu=False):
    """Same per-element order as Fig. 9 (ct, kj, ki, ifm), vectorised over the
    non-reduction dims; float64."""
    n, ct, h, wd, _ = x.shape
    kt, _, r, s, _, _ = w.shape
    p, q = out_hw(h, wd, r, s, stride, pad)
    xp = pad_nchw16c(x, r, s, stride, pad).astype(np.float64)
    wd64 = w.astype(np.float64)
    y = np.zeros((n, kt, p, q, 16))
    for c in range(ct):
        for kj in range(r):
            for ki in range(s):
                patch = xp[:, c, kj:kj + stride * (p - 1) + 1:stride,
                           ki:ki + stride * (q - 1) + 1:stride, :]  # n,p,q,ifm
                for ifm in range(16):
                    # y[n,kt,p,q,ofm] += w[kt,c,kj,ki,ifm,ofm] * x[n,p,q,ifm]
                    y += (wd64[:, c, kj, ki, ifm, :][None, :, None, None, :]
                          * patch[:, None, :, :, ifm, None])
    if bias is not None:
        y = y + np.asarray(bias, np.float64).reshape(1, kt, 1, 1, 16)
    if relu:
        y = np.where(0.0 > y, 0.0, y)
    return y


def gemm_np(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    c = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        c = c + a[:, k:k + 1] * b[k:k + 1, :]
    return c
