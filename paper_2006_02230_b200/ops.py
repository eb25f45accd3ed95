"""Torch-facing ops over the C ABI.  torch supplies device memory and the
current CUDA stream; all arithmetic runs in libpdl.so kernels.

Layouts (the reference nest's array declarations):
  x  [N][C/16][H][W][16]          nChw16c activations, UNPADDED
     [N][H][W][4]                 compact narrow-channel input (C <= 4, the ResNet stem):
                                  a 4-D x selects PDL_X_NCHW4C (to_nchw4c() makes it)
  w  [K/16][C/16][R][S][16c][16k]  KCRS16c16k weights
  y  [N][K/16][P][Q][16]           nKhw16k outputs
  bias [K]
"""
from __future__ import annotations

import contextlib
import ctypes
import warnings
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (PDL_BIAS, PDL_HOST_X_READY, PDL_MODE_FP32, PDL_NO_SIMT, PDL_OP_GEMM, PDL_RELU,
                   PDL_RELU6, PDL_SCALE, PDL_X_NCHW4C, MODES, TileCfg, check, lib)


class SimtPathWarning(UserWarning):
    """A tensor-core-mode GEMM ran on the CUDA cores (exact fp32) because TMA
    cannot describe its operands (N or K not a multiple of 4, unaligned views)."""


def _mode(mode: str) -> int:
    try:
        return MODES[mode.lower()]
    except KeyError:
        raise ValueError(f"unknown mode {mode!r}; expected one of {sorted(MODES)}") from None


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _on(stream):
    """Allocate (and zero) temporaries on the stream the library call runs on: the
    caching allocator then reuses their blocks only in that stream's order, so a
    temporary freed when the Python call returns is never handed out while a
    kernel on `stream` may still read it."""
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need_cuda_f32(name, t):
    if t is None:
        return
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _cfg_ptr(cfg):
    if cfg is None:
        return None
    if isinstance(cfg, dict):
        cfg = TileCfg.make(**cfg)
    return ctypes.byref(cfg)


_split_ws: dict = {}
_split_ws_retired: list = []


def _split_workspace(device, stream_handle: int, nbytes: int):
    """Zero-initialised split-K workspace, one per (device, stream): its tile
    counters reset themselves at the end of every launch, so concurrent streams
    must not share one.  Buffers are only ever added (a CUDA graph captured
    earlier keeps pointing at the old one), growing 2x at a time.  Called under
    `_on(stream)`: the zero fill is ordered before the kernels that use it."""
    if nbytes == 0:
        return None
    key = (torch.device(device).index, stream_handle)
    ws = _split_ws.get(key)
    if ws is None or ws.numel() * 4 < nbytes:
        if ws is not None:
            _split_ws_retired.append(ws)
            nbytes = max(nbytes, ws.numel() * 8)
        ws = torch.zeros((nbytes + 3) // 4, dtype=torch.float32, device=device)
        _split_ws[key] = ws
    return ws


def conv_out_hw(h, w, r, s, stride, pad):
    return (h + 2 * pad - r) // stride + 1, (w + 2 * pad - s) // stride + 1


@dataclass
class PackedWeights:
    """Tensor-core operand image of KCRS16c16k weights (hi/lo planes for 3xTF32)."""
    data: torch.Tensor
    C: int
    K: int
    R: int
    S: int
    mode: str


def prepack_weights(w: torch.Tensor, mode: str = "3xtf32", channels: int | None = None,
                    stream=None) -> PackedWeights:
    """One-time reorder of KCRS16c16k weights into the tensor-core operand image.
    `channels` = true input channels C when the last 16-block is padded (the
    ResNet stem has C=3 stored in one 16-channel block)."""
    _need_cuda_f32("w", w)
    kt, ct, r, s, c16, k16 = w.shape
    assert c16 == 16 and k16 == 16, "weights must be KCRS16c16k"
    C, K = (channels if channels is not None else ct * 16), kt * 16
    if not (ct * 16 - 16 < C <= ct * 16):
        raise ValueError(f"channels={C} inconsistent with {ct} channel blocks")
    flags = _mode(mode)
    nbytes = lib().pdl_conv2d_packed_bytes(C, K, r, s, flags)
    out = torch.empty(nbytes // 4, dtype=torch.float32, device=w.device)
    check(lib().pdl_conv2d_prepack_weights(_ptr(w), _ptr(out), C, K, r, s, flags,
                                           ctypes.c_void_p(_stream(stream))))
    return PackedWeights(out, C, K, r, s, mode.lower())


def _epilogue(bias, relu: bool, relu6: bool, scale, K: int):
    """Epilogue flags and the device buffer the kernels read them from: `bias`
    alone, or [shift[K] | scale[K]] when a per-channel scale is fused (PDL_SCALE)."""
    _need_cuda_f32("bias", bias)
    _need_cuda_f32("scale", scale)
    flags = (PDL_BIAS if bias is not None else 0) | (PDL_RELU if relu else 0) | \
        (PDL_RELU6 if relu6 else 0)
    buf = bias
    if scale is not None:
        if scale.numel() != K or (bias is not None and bias.numel() != K):
            raise ValueError(f"scale / bias must hold K={K} values")
        shift = bias.reshape(-1) if bias is not None else torch.zeros(K, device=scale.device)
        buf = torch.cat([shift, scale.reshape(-1)])
        flags |= PDL_SCALE
    return flags, buf


def conv2d_nchw16c(x: torch.Tensor, w, bias: torch.Tensor | None = None, stride: int = 1,
                   pad: int = 0, relu: bool = False, mode: str = "3xtf32", cfg=None,
                   out: torch.Tensor | None = None, channels: int | None = None,
                   stream=None, relu6: bool = False, scale: torch.Tensor | None = None) -> torch.Tensor:
    """Blocked conv fwd with the fused epilogue y = act(conv * scale[k] + bias[k]),
    act = ReLU (relu=True) or ReLU6 (relu6=True); scale (batch-norm inference
    affine) and bias optional.  `w` is either raw KCRS16c16k weights or a
    PackedWeights from prepack_weights().  `channels` = true input channels when
    x's last 16-channel block is zero-padded (C <= 4 selects the narrow stem
    kernel)."""
    _need_cuda_f32("x", x)
    _need_cuda_f32("bias", bias)
    n, ct, h, wd, compact = _x_dims(x)
    packed = w if isinstance(w, PackedWeights) else None
    if packed is not None:
        C, K, R, S = packed.C, packed.K, packed.R, packed.S
        if packed.mode != mode.lower():
            raise ValueError(f"weights packed for {packed.mode}, called with {mode}")
    else:
        _need_cuda_f32("w", w)
        kt, ct2, R, S, _, _ = w.shape
        C, K = (channels if channels is not None else ct2 * 16), kt * 16
    if channels is not None and channels != C:
        raise ValueError(f"channels={channels} but weights were packed for C={C}")
    if not (ct * 16 - 16 < C <= ct * 16):
        raise ValueError(f"channel mismatch: x has {ct} blocks of 16, w has C={C}")
    if compact and C > 4:
        raise ValueError(f"a 4-D x is the compact [N][H][W][4] layout (C <= 4); weights have C={C}")
    P, Q = conv_out_hw(h, wd, R, S, stride, pad)
    with _on(stream):
        return _conv2d_call(x, w, packed, bias, out, n, C, K, h, wd, R, S, P, Q, stride, pad, relu,
                            relu6, scale, mode, cfg, stream, PDL_X_NCHW4C if compact else 0)


def _x_dims(x):
    """(N, channel blocks, H, W, compact) of a conv input: 5-D nChw16c, or the 4-D
    compact [N][H][W][4] layout of the narrow-channel path."""
    if x.dim() == 4:
        n, h, wd, v = x.shape
        if v != 4:
            raise ValueError("a 4-D x must be [N][H][W][4] (compact narrow-channel layout)")
        return n, 1, h, wd, True
    n, ct, h, wd, v = x.shape
    if v != 16:
        raise ValueError("x must be nChw16c")
    return n, ct, h, wd, False


def _conv2d_call(x, w, packed, bias, out, n, C, K, h, wd, R, S, P, Q, stride, pad, relu, relu6,
                 scale, mode, cfg, stream, xflags=0):
    y = out if out is not None else torch.empty((n, K // 16, P, Q, 16), dtype=torch.float32,
                                                device=x.device)
    _need_cuda_f32("out", y)
    eflags, bias = _epilogue(bias, relu, relu6, scale, K)
    flags = _mode(mode) | eflags | xflags
    st = ctypes.c_void_p(_stream(stream))
    cp = _cfg_ptr(cfg)
    if packed is not None:
        # split-K (tiles that leave SMs idle, e.g. 7x7 maps at small batches) needs a workspace
        need = lib().pdl_conv2d_splitk_workspace_bytes(n, C, K, h, wd, R, S, stride, pad, flags, cp)
        ws = _split_workspace(x.device, st.value or 0, need)
        check(lib().pdl_conv2d_fwd_prepacked_ws(_ptr(x), _ptr(packed.data), _ptr(bias), _ptr(y), n,
                                                C, K, h, wd, R, S, stride, pad, flags, cp, _ptr(ws),
                                                need, st))
    else:
        nbytes = lib().pdl_conv2d_packed_bytes(C, K, R, S, flags)
        split = lib().pdl_conv2d_splitk_workspace_bytes(n, C, K, h, wd, R, S, stride, pad, flags, cp)
        off = (nbytes + 255) // 256 * 256
        total = off + split if split else nbytes
        ws = torch.empty(max((total + 3) // 4, 4), dtype=torch.float32, device=x.device)
        if split:  # fresh buffer: the split-K tile counters must start at zero
            ws.view(torch.uint8)[off:].zero_()
        check(lib().pdl_conv2d_fwd_nchw16c(_ptr(x), _ptr(w), _ptr(bias), _ptr(y), n, C, K, h, wd,
                                           R, S, stride, pad, flags, cp, _ptr(ws), total, st))
    return y


_host_ws: dict = {}


def _host_workspace(device, stream_handle: int, nbytes: int) -> torch.Tensor:
    """Device staging for conv2d_nchw16c_host, kept per (device, stream) and grown
    on demand: calls on one stream are ordered (each joins its copy streams back
    into the caller's stream), calls on different streams must not share it."""
    key = (torch.device(device).index, stream_handle)
    ws = _host_ws.get(key)
    if ws is None or ws.numel() * 4 < nbytes:
        ws = torch.empty((nbytes + 3) // 4, dtype=torch.float32, device=device)
        _host_ws[key] = ws
    return ws


def conv2d_nchw16c_host(x: torch.Tensor, w: PackedWeights, bias: torch.Tensor | None = None,
                        stride: int = 1, pad: int = 0, relu: bool = False, mode: str = "3xtf32",
                        cfg=None, out: torch.Tensor | None = None, chunk: int = 0,
                        device=None, stream=None, x_ready: bool = False, relu6: bool = False,
                        scale: torch.Tensor | None = None) -> torch.Tensor:
    """Blocked conv fwd over HOST buffers (the reference's interpret() contract:
    host arrays in, host array out).  x / out are CPU float32 tensors -- pinned
    for full PCIe speed -- weights (PackedWeights) and bias live on the GPU.  The
    library pipelines image chunks: H2D copy, fused conv and D2H copy overlap
    (pdl_conv2d_fwd_host).  Returns `out` (allocated pinned if None), complete
    once `stream` reaches the point after this call.  x_ready=True promises that
    x, the packed weights and bias are not written by work still pending on
    `stream` (e.g. x is not the output of an earlier host call): this call's
    copies in and convolutions may then overlap the previous call's copies out
    (PDL_HOST_X_READY)."""
    if not isinstance(w, PackedWeights):
        raise TypeError("conv2d_nchw16c_host takes PackedWeights (prepack_weights())")
    if not isinstance(x, torch.Tensor) or x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError("x must be a contiguous float32 CPU tensor")
    _need_cuda_f32("bias", bias)
    if w.mode != mode.lower():
        raise ValueError(f"weights packed for {w.mode}, called with {mode}")
    n, ct, h, wd, compact = _x_dims(x)
    if not (ct * 16 - 16 < w.C <= ct * 16) or (compact and w.C > 4):
        raise ValueError(f"x must be nChw16c (or, for C <= 4, [N][H][W][4]) with {w.C} channels")
    P, Q = conv_out_hw(h, wd, w.R, w.S, stride, pad)
    y = out if out is not None else torch.empty((n, w.K // 16, P, Q, 16), dtype=torch.float32,
                                                pin_memory=True)
    if y.is_cuda or y.dtype != torch.float32 or not y.is_contiguous() or \
            tuple(y.shape) != (n, w.K // 16, P, Q, 16):
        raise ValueError("out must be a contiguous float32 CPU tensor [N][K/16][P][Q][16]")
    dev = w.data.device if device is None else torch.device(device)
    need = lib().pdl_conv2d_host_workspace_bytes(n, w.C, w.K, h, wd, w.R, w.S, stride, pad, chunk)
    sh = _stream(stream)
    ws = _host_workspace(dev, sh, need)
    with _on(stream):
        eflags, bias = _epilogue(bias, relu, relu6, scale, w.K)
    flags = _mode(mode) | eflags | (PDL_X_NCHW4C if compact else 0)
    if x_ready and scale is None:   # (a fused scale builds its [shift | scale] buffer on `stream`)
        flags |= PDL_HOST_X_READY
    check(lib().pdl_conv2d_fwd_host(_ptr(x), _ptr(w.data), _ptr(bias), _ptr(y), n, w.C, w.K, h, wd,
                                    w.R, w.S, stride, pad, flags, _cfg_ptr(cfg), int(chunk),
                                    _ptr(ws), ws.numel() * 4, ctypes.c_void_p(sh)))
    return y


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor | None = None, alpha: float = 1.0,
         beta: float = 0.0, relu: bool = False, mode: str = "3xtf32", cfg=None,
         stream=None, relu6: bool = False, bias: torch.Tensor | None = None,
         scale: torch.Tensor | None = None, strict: bool = False) -> torch.Tensor:
    """C = act((alpha * A @ B + beta * C) * scale[n] + bias[n]) (row-major fp32), act =
    ReLU / ReLU6 / none, scale and bias optional (the fused GEMM epilogue of Alg. 3,
    PAPER.md:1228-1241).  Shapes the tensor cores cannot take through TMA (N or K not
    a multiple of 4) run on the CUDA cores in exact fp32 with a SimtPathWarning;
    strict=True raises instead."""
    for nm, t in (("a", a), ("b", b)):
        _need_cuda_f32(nm, t)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    with _on(stream):
        if c is None:
            if beta != 0.0:
                raise ValueError("beta != 0 needs c")
            c = torch.empty((m, n), dtype=torch.float32, device=a.device)
        _need_cuda_f32("c", c)
        eflags, ebuf = _epilogue(bias, relu, relu6, scale, n)
        flags = _mode(mode) | eflags
        if (flags & 0x30) != PDL_MODE_FP32 and m and n and not (
                k > 0 and n % 4 == 0 and k % 4 == 0 and
                all(t.data_ptr() % 16 == 0 for t in (a, b, c))):
            if strict:
                flags |= PDL_NO_SIMT
            else:
                warnings.warn(f"gemm {m}x{n}x{k}: operands not TMA-describable, running the exact-fp32 "
                              "CUDA-core kernel", SimtPathWarning, stacklevel=2)
        cp = _cfg_ptr(cfg)
        sh = _stream(stream)
        dims = (ctypes.c_int * 4)(m, n, k, flags)
        need = lib().pdl_workspace_bytes(PDL_OP_GEMM, dims, cp)
        ws = _split_workspace(a.device, sh, need)
        check(lib().pdl_gemm_f32_epilogue(_ptr(a), _ptr(b), _ptr(c), _ptr(ebuf), m, n, k, k, n, n,
                                          float(alpha), float(beta), flags, cp, _ptr(ws), need,
                                          ctypes.c_void_p(sh)))
    return c


def bias_relu_(y: torch.Tensor, bias: torch.Tensor | None, relu: bool = True,
               stream=None, relu6: bool = False, scale: torch.Tensor | None = None) -> torch.Tensor:
    """Unfused element-wise pass y = act(y * scale + bias) in place over nKhw16k (the
    GPU baseline of the fused epilogue, and the stand-alone element-wise nest)."""
    _need_cuda_f32("y", y)
    n, kt, p, q, v = y.shape
    with _on(stream):
        flags, bias = _epilogue(bias, relu, relu6, scale, kt * 16)
        check(lib().pdl_bias_relu_nchw16c(_ptr(y), _ptr(bias), n, kt * 16, p, q, flags,
                                          ctypes.c_void_p(_stream(stream))))
    return y


def accumulate_(y: torch.Tensor, y0: torch.Tensor, bias: torch.Tensor | None = None,
                relu: bool = False, stream=None, relu6: bool = False,
                scale: torch.Tensor | None = None) -> torch.Tensor:
    """y = act((y + y0) * scale + bias) in place over nKhw16k: a convolution's `+=`
    onto incoming output contents y0, with the nest's element-wise epilogue."""
    _need_cuda_f32("y", y)
    _need_cuda_f32("y0", y0)
    if y0.shape != y.shape:
        raise ValueError(f"y0 {tuple(y0.shape)} != y {tuple(y.shape)}")
    n, kt, p, q, v = y.shape
    with _on(stream):
        flags, bias = _epilogue(bias, relu, relu6, scale, kt * 16)
        check(lib().pdl_accumulate_epilogue_nchw16c(_ptr(y), _ptr(y0), _ptr(bias), n, kt * 16, p, q,
                                                    flags, ctypes.c_void_p(_stream(stream))))
    return y


def to_nchw16c(x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """NCHW -> nChw16c (channels padded with zeros to a multiple of 16)."""
    x = x.contiguous()
    _need_cuda_f32("x", x)
    n, c, h, w = x.shape
    if out is None:
        out = torch.empty((n, (c + 15) // 16, h, w, 16), dtype=torch.float32, device=x.device)
    check(lib().pdl_pack_nchw16c(_ptr(x), _ptr(out), n, c, h, w, ctypes.c_void_p(_stream(stream))))
    return out


def to_nchw4c(x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """NCHW with C <= 4 -> the compact [N][H][W][4] input of the narrow-channel conv
    (channels >= C zero); conv2d_nchw16c / conv2d_nchw16c_host take it as a 4-D x."""
    x = x.contiguous()
    _need_cuda_f32("x", x)
    n, c, h, w = x.shape
    if c > 4:
        raise ValueError(f"to_nchw4c: C must be <= 4, got {c}")
    if out is None:
        out = torch.empty((n, h, w, 4), dtype=torch.float32, device=x.device)
    check(lib().pdl_pack_nchw4c(_ptr(x), _ptr(out), n, c, h, w, ctypes.c_void_p(_stream(stream))))
    return out


def from_nchw16c(y: torch.Tensor, channels: int | None = None, out: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """nChw16c -> NCHW, dropping padding channels beyond `channels`."""
    _need_cuda_f32("y", y)
    n, cb, h, w, v = y.shape
    c = channels if channels is not None else cb * 16
    if out is None:
        out = torch.empty((n, c, h, w), dtype=torch.float32, device=y.device)
    check(lib().pdl_unpack_nchw16c(_ptr(y), _ptr(out), n, c, h, w, ctypes.c_void_p(_stream(stream))))
    return out


def weights_to_kcrs16c16k(w: torch.Tensor, stream=None) -> torch.Tensor:
    """OIHW [K][C][R][S] -> KCRS16c16k (input channels padded with zeros)."""
    w = w.contiguous()
    _need_cuda_f32("w", w)
    k, c, r, s = w.shape
    out = torch.empty((k // 16, (c + 15) // 16, r, s, 16, 16), dtype=torch.float32, device=w.device)
    check(lib().pdl_pack_kcrs16c16k(_ptr(w), _ptr(out), k, c, r, s, ctypes.c_void_p(_stream(stream))))
    return out


def conv2d_nchw(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, stride: int = 1,
                pad: int = 0, relu: bool = False, mode: str = "3xtf32", cfg=None,
                stream=None) -> torch.Tensor:
    """PyTorch-layout convenience: NCHW x, OIHW w -> NCHW y, through pack ->
    blocked conv (+bias, +ReLU) -> unpack; all on the GPU."""
    c = x.shape[1]
    with _on(stream):   # the intermediates xb / pw / yb live (and die) on `stream`
        xb = to_nchw16c(x, stream=stream)
        pw = prepack_weights(weights_to_kcrs16c16k(w, stream=stream), mode=mode, channels=c,
                             stream=stream)
        yb = conv2d_nchw16c(xb, pw, bias, stride=stride, pad=pad, relu=relu, mode=mode, cfg=cfg,
                            channels=c, stream=stream)
        return from_nchw16c(yb, w.shape[0], stream=stream)


def device_ok() -> bool:
    return lib().pdl_device_check() == 0


__all__ = ["conv2d_nchw16c", "prepack_weights", "PackedWeights", "gemm", "bias_relu_", "accumulate_",
           "device_ok", "conv_out_hw", "TileCfg", "SimtPathWarning", "to_nchw4c"]
_ = _lib
