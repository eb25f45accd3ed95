"""ctypes binding of libpdl.so (include/pdl.h).

The product path has no CPU fallback: if the library is missing or the device
is not an sm_100 B200, every op raises `PdlError` / `PdlDeviceError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
# PDL_LIB: load another build of the library (A/B experiments between builds)
LIB_PATH = os.environ.get("PDL_LIB") or os.path.join(_PKG, "libpdl.so")

PDL_BIAS = 1
PDL_RELU = 2
PDL_RELU6 = 1 << 2
PDL_SCALE = 1 << 3
PDL_MODE_3XTF32 = 0 << 4
PDL_MODE_TF32 = 1 << 4
PDL_MODE_FP32 = 2 << 4
PDL_MODE_MASK = 3 << 4
PDL_HOST_X_READY = 1 << 6
PDL_NO_SIMT = 1 << 7
PDL_X_NCHW4C = 1 << 13
PDL_OP_CONV2D = 1
PDL_OP_GEMM = 2

MODES = {"3xtf32": PDL_MODE_3XTF32, "tf32": PDL_MODE_TF32, "fp32": PDL_MODE_FP32}

PDL_OK, PDL_EINVAL, PDL_EALIGN, PDL_EDEVICE, PDL_ELAUNCH, PDL_EWORKSPACE, PDL_EUNSUPPORTED = (
    0, -1, -2, -3, -4, -5, -6)

# Symbols include/pdl.h declares (checked by tests/test_capi.py without a GPU).
EXPORTS = (
    "pdl_conv2d_fwd_nchw16c", "pdl_conv2d_packed_bytes", "pdl_conv2d_prepack_weights",
    "pdl_conv2d_fwd_prepacked", "pdl_gemm_f32", "pdl_bias_relu_nchw16c",
    "pdl_workspace_bytes", "pdl_default_cfg", "pdl_last_launch_count", "pdl_last_error",
    "pdl_abi_version", "pdl_device_check", "pdl_pack_nchw16c", "pdl_unpack_nchw16c",
    "pdl_pack_kcrs16c16k", "pdl_conv2d_host_workspace_bytes", "pdl_conv2d_fwd_host",
    "pdl_conv2d_splitk_workspace_bytes", "pdl_conv2d_fwd_prepacked_ws", "pdl_gemm_f32_epilogue",
    "pdl_accumulate_epilogue_nchw16c", "pdl_conv2d_schedule", "pdl_gemm_schedule", "pdl_pack_nchw4c",
)


class PdlError(RuntimeError):
    """A libpdl call returned a nonzero status (message from pdl_last_error)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class PdlDeviceError(PdlError):
    pass


class PdlShapeError(PdlError, ValueError):
    pass


class TileCfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("bm", "bn", "bk", "stages", "cluster_m", "cluster_n", "split_k", "raster")]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}

    @classmethod
    def make(cls, **kw) -> "TileCfg":
        c = cls()
        for k, v in kw.items():
            setattr(c, k, int(v))
        return c


class Schedule(ctypes.Structure):
    """pdl_schedule (include/pdl.h): the schedule the library will actually run."""
    _fields_ = [(n, ctypes.c_int) for n in
                ("kind", "bn", "bk", "cluster", "tile_w", "tile_h", "tile_images", "seg_rows",
                 "m_tiles", "n_tiles", "num_kb", "split", "kb_per", "halo", "resident", "pair",
                 "order", "flat")] + [("splitk_workspace_bytes", ctypes.c_size_t)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


_lock = threading.Lock()
_lib = None

_vp = ctypes.c_void_p
_i = ctypes.c_int
_u = ctypes.c_uint
_sz = ctypes.c_size_t


# Entry points an older build may lack (PDL_LIB A/B runs against a previous round's
# library): declared only when present.
_OPTIONAL = ("pdl_gemm_f32_epilogue", "pdl_accumulate_epilogue_nchw16c", "pdl_conv2d_schedule",
             "pdl_gemm_schedule", "pdl_pack_nchw4c")


class _Skip:
    """Stand-in for a missing optional symbol while declaring (attribute writes vanish)."""
    def __setattr__(self, k, v):
        pass


class _Tolerant:
    def __init__(self, L):
        object.__setattr__(self, "_L", L)

    def __getattr__(self, name):
        try:
            return getattr(self._L, name)
        except AttributeError:
            if name in _OPTIONAL and os.environ.get("PDL_LIB"):
                return _Skip()
            raise


def _declare(L):
    L = _Tolerant(L)
    L.pdl_conv2d_fwd_nchw16c.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 9 + [
        _u, ctypes.POINTER(TileCfg), _vp, _sz, _vp]
    L.pdl_conv2d_packed_bytes.argtypes = [_i, _i, _i, _i, _u]
    L.pdl_conv2d_packed_bytes.restype = _sz
    L.pdl_conv2d_prepack_weights.argtypes = [_vp, _vp, _i, _i, _i, _i, _u, _vp]
    L.pdl_conv2d_fwd_prepacked.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 9 + [
        _u, ctypes.POINTER(TileCfg), _vp]
    L.pdl_conv2d_splitk_workspace_bytes.argtypes = [_i] * 9 + [_u, ctypes.POINTER(TileCfg)]
    L.pdl_conv2d_splitk_workspace_bytes.restype = _sz
    L.pdl_conv2d_fwd_prepacked_ws.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 9 + [
        _u, ctypes.POINTER(TileCfg), _vp, _sz, _vp]
    L.pdl_conv2d_host_workspace_bytes.argtypes = [_i] * 10
    L.pdl_conv2d_host_workspace_bytes.restype = _sz
    L.pdl_conv2d_fwd_host.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 9 + [
        _u, ctypes.POINTER(TileCfg), _i, _vp, _sz, _vp]
    L.pdl_gemm_f32.argtypes = [_vp, _vp, _vp] + [_i] * 6 + [
        ctypes.c_float, ctypes.c_float, _u, ctypes.POINTER(TileCfg), _vp, _sz, _vp]
    L.pdl_gemm_f32_epilogue.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 6 + [
        ctypes.c_float, ctypes.c_float, _u, ctypes.POINTER(TileCfg), _vp, _sz, _vp]
    L.pdl_bias_relu_nchw16c.argtypes = [_vp, _vp, _i, _i, _i, _i, _u, _vp]
    L.pdl_accumulate_epilogue_nchw16c.argtypes = [_vp, _vp, _vp, _i, _i, _i, _i, _u, _vp]
    L.pdl_conv2d_schedule.argtypes = [_i] * 9 + [_u, ctypes.POINTER(TileCfg), _i, ctypes.POINTER(Schedule)]
    L.pdl_gemm_schedule.argtypes = [_i, _i, _i, _u, ctypes.POINTER(TileCfg), _i, ctypes.POINTER(Schedule)]
    L.pdl_pack_nchw16c.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp]
    L.pdl_pack_nchw4c.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp]
    L.pdl_unpack_nchw16c.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp]
    L.pdl_pack_kcrs16c16k.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp]
    L.pdl_workspace_bytes.argtypes = [_i, ctypes.POINTER(_i), ctypes.POINTER(TileCfg)]
    L.pdl_workspace_bytes.restype = _sz
    L.pdl_default_cfg.argtypes = [_i, ctypes.POINTER(_i), ctypes.POINTER(TileCfg)]
    L.pdl_last_launch_count.argtypes = []
    L.pdl_last_error.argtypes = []
    L.pdl_last_error.restype = ctypes.c_char_p
    L.pdl_abi_version.argtypes = []
    L.pdl_device_check.argtypes = []
    for name in EXPORTS:
        if name not in ("pdl_conv2d_packed_bytes", "pdl_workspace_bytes", "pdl_last_error",
                        "pdl_conv2d_host_workspace_bytes", "pdl_conv2d_splitk_workspace_bytes"):
            getattr(L, name).restype = _i


def lib():
    """Load libpdl.so once; raise if it was not built (no silent fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise PdlError(PDL_EDEVICE, f"{LIB_PATH} is missing: run "
                                   "`python -c 'import __graft_entry__ as g; g.build()'`")
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == PDL_OK:
        return
    msg = lib().pdl_last_error().decode(errors="replace")
    if rc == PDL_EDEVICE:
        raise PdlDeviceError(rc, msg)
    if rc in (PDL_EINVAL, PDL_EALIGN, PDL_EUNSUPPORTED, PDL_EWORKSPACE):
        raise PdlShapeError(rc, msg)
    raise PdlError(rc, msg)


def default_cfg(op: int, dims) -> TileCfg:
    arr = (_i * len(dims))(*[int(d) for d in dims])
    c = TileCfg()
    check(lib().pdl_default_cfg(op, arr, ctypes.byref(c)))
    return c


def conv_schedule(N, C, K, H, W, R, S, stride, pad, flags, cfg=None, with_workspace=True) -> dict:
    """The schedule libpdl runs for this conv call (host-only; works without a GPU)."""
    out = Schedule()
    cp = None if cfg is None else ctypes.byref(cfg if isinstance(cfg, TileCfg) else TileCfg.make(**cfg))
    check(lib().pdl_conv2d_schedule(N, C, K, H, W, R, S, stride, pad, flags, cp, int(with_workspace),
                                    ctypes.byref(out)))
    return out.as_dict()


def gemm_schedule(M, N, K, flags, cfg=None, with_workspace=True) -> dict:
    out = Schedule()
    cp = None if cfg is None else ctypes.byref(cfg if isinstance(cfg, TileCfg) else TileCfg.make(**cfg))
    check(lib().pdl_gemm_schedule(M, N, K, flags, cp, int(with_workspace), ctypes.byref(out)))
    return out.as_dict()


def last_launch_count() -> int:
    return int(lib().pdl_last_launch_count())
