"""One small launch per kernel family of libpdl.so (stem, halo, resident weights,
stride-2 parity maps, per-tap boxes, split-K, segment tiles, multicast clusters,
TF32 SS / 256-column tiles, extended epilogue, GEMM TS / SS / split-K / bias, the
CUDA-core kernels, the host pipeline, layout and element-wise kernels).

Each family runs the product path through the C ABI on a small shape and checks
  * the result against the CPU oracle,
  * guard bands (canaries) on both sides of the output buffer: an out-of-bounds
    store of any epilogue path lands there,
  * a second launch into a fresh buffer is bitwise equal (a race between the
    pipeline roles shows up as run-to-run differences).
It is also the target for compute-sanitizer where that tool is allowed:
    compute-sanitizer --tool memcheck|synccheck|racecheck python scripts/sanitize_case.py FAMILY...
(`all` = every family).  Used by tests/test_gpu_sanitizer.py and scripts/gpu_sanitize.sh.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2006_02230_b200 as P  # noqa: E402
from paper_2006_02230_b200 import _lib, workloads as W  # noqa: E402


CANARY = -12345.0


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def conv_case(C, K, H, R, stride, N, mode="3xtf32", cfg=None, tol=1e-5, expect=None, **epi):
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=11)
    flags = _lib.MODES[mode] | 3
    if expect:
        c = None if cfg is None else _lib.TileCfg.make(**cfg)
        s = _lib.conv_schedule(N, C, K, H, H, R, R, stride, R // 2, flags, c)
        for k, v in expect.items():
            assert s[k] == v, f"schedule {k}={s[k]}, the case wants {v}: {s}"
    wd = torch.from_numpy(w).cuda()
    # exact-fp32 mode takes raw weights (no tensor-core operand image)
    pw = wd if mode == "fp32" else P.prepack_weights(wd, mode=mode, channels=C)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = {}
    ref_kw = {}
    # guard bands around y: an out-of-bounds store of the epilogue (TMA box or direct)
    # lands in the canaries
    P_, Q_ = P.conv_out_hw(H, H, R, R, stride, R // 2)
    ny = N * K * P_ * Q_
    guard = 4096
    ybuf = torch.full((ny + 2 * guard,), CANARY, dtype=torch.float32, device="cuda")
    kw["out"] = ybuf[guard:guard + ny].view(N, K // 16, P_, Q_, 16)
    if epi.get("scale"):
        sc = np.linspace(0.5, 1.5, K).astype(np.float32)
        kw.update(scale=torch.from_numpy(sc).cuda(), relu6=True)
        y = P.conv2d_nchw16c(xd, pw, bd, stride=stride, pad=R // 2, mode=mode, cfg=cfg, channels=C, **kw)
        ref = oracle.conv2d_f64(x, w, None, stride=stride, pad=R // 2, relu=False)
        kt = np.arange(K).reshape(K // 16, 16)
        ref = ref * sc.astype(np.float64)[kt][None, :, None, None, :] + \
            b.astype(np.float64)[kt][None, :, None, None, :]
        ref = np.minimum(np.maximum(ref, 0.0), 6.0)
    else:
        y = P.conv2d_nchw16c(xd, pw, bd, stride=stride, pad=R // 2, relu=True, mode=mode, cfg=cfg,
                             channels=C, **kw)
        ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True, **ref_kw)
    torch.cuda.synchronize()
    assert bool((ybuf[:guard] == CANARY).all()) and bool((ybuf[guard + ny:] == CANARY).all()), \
        "conv wrote outside y"
    kw.pop("out")
    y_again = P.conv2d_nchw16c(xd, pw, bd, stride=stride, pad=R // 2, relu=not epi.get("scale"),
                               mode=mode, cfg=cfg, channels=C, **kw)
    assert torch.equal(y, y_again), "two launches differ bitwise"
    e = rel(y.cpu().numpy(), ref)
    assert e <= tol, f"max-rel {e:.3e} > {tol}"
    return e


def gemm_case(m, n, k, mode="3xtf32", cfg=None, tol=1e-5, bias=False):
    a, b = W.gemm_inputs(m, n, k, seed=4)
    kw = {}
    ref = oracle.gemm_f64(a, b)
    if bias:
        bv = np.linspace(-1, 1, n).astype(np.float32)
        kw.update(bias=torch.from_numpy(bv).cuda(), relu=True)
        ref = np.maximum(ref + bv.astype(np.float64)[None, :], 0.0)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", P.SimtPathWarning)
        guard = 4096
        cbuf = torch.full((m * n + 2 * guard,), CANARY, dtype=torch.float32, device="cuda")
        c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                   c=cbuf[guard:guard + m * n].view(m, n), mode=mode, cfg=cfg, **kw)
    torch.cuda.synchronize()
    assert bool((cbuf[:guard] == CANARY).all()) and bool((cbuf[guard + m * n:] == CANARY).all()), \
        "gemm wrote outside C"
    e = rel(c.cpu().numpy(), ref)
    assert e <= tol, f"max-rel {e:.3e} > {tol}"
    return e


def fam_stem():
    return conv_case(3, 64, 40, 7, 2, 2, expect={"kind": 2})


def fam_stem_tf32():
    return conv_case(3, 64, 40, 7, 2, 1, mode="tf32", tol=1e-2, expect={"kind": 2})


def fam_halo():
    return conv_case(128, 128, 28, 3, 1, 2, cfg={"split_k": 1}, expect={"halo": 1, "split": 1})


def fam_halo_cg4():
    return conv_case(64, 64, 28, 3, 1, 2, expect={"halo": 1, "bk": 64})


def fam_halo_splitk():
    return conv_case(256, 256, 14, 3, 1, 1, cfg={"split_k": 3}, expect={"halo": 1, "split": 3})


def fam_resident():
    return conv_case(64, 256, 28, 1, 1, 2, expect={"resident": 1})


def fam_stride2():
    return conv_case(256, 128, 28, 1, 2, 2, expect={"resident": 0, "halo": 0})


def fam_pertap():
    return conv_case(128, 128, 14, 3, 2, 2, expect={"halo": 0})


def fam_splitk():
    return conv_case(1024, 256, 7, 1, 1, 2, cfg={"split_k": 4}, expect={"split": 4})


def fam_segtiles():
    return conv_case(256, 256, 14, 1, 1, 5, cfg={"raster": 4}, expect={"seg_rows": 9})


def _tile(bw, bh, bni):
    return {"raster": bw << 8 | bh << 16 | bni << 24}  # PDL_RASTER_TILE


def fam_multibox_ragged():
    # 7x1 pixels x 18 images per tile, 37 images: the last boxes hold images past N (TMA clips the stores)
    return conv_case(256, 128, 14, 1, 2, 37, cfg=_tile(7, 1, 18), expect={"tile_w": 7, "tile_h": 1, "tile_images": 18})


def fam_multibox_halo():
    # 8x8 pixels x 2 images per tile with the halo path, odd batch
    return conv_case(64, 64, 56, 3, 1, 5, cfg=_tile(8, 8, 2), expect={"tile_w": 8, "tile_h": 8, "tile_images": 2, "halo": 1})


def fam_multibox_1x1():
    # 7x7 1x1, rows of 18 images, 23 images
    return conv_case(256, 256, 7, 1, 1, 23, cfg=_tile(7, 1, 18), expect={"tile_w": 7, "tile_images": 18, "flat": 0})


def fam_multibox_splitk():
    # 7x7 3x3 at a small batch: 7x1 x 18 images, per-tap boxes, two split-K ranges (register fast path)
    return conv_case(512, 512, 7, 3, 1, 32, expect={"tile_images": 18, "split": 2})


def fam_3xtf32_bn256():
    # 256-column 3xTF32 tiles: single accumulator, register-traded epilogue, ragged batch and channels
    return conv_case(256, 384, 14, 1, 1, 11, cfg={"bn": 256, "bk": 32}, expect={"bn": 256})


def fam_cluster():
    return conv_case(256, 256, 14, 1, 1, 4, cfg={"cluster_m": 2}, expect={"cluster": 2})


def fam_tf32():
    return conv_case(128, 128, 14, 1, 1, 2, mode="tf32", tol=1e-2)


def fam_tf32_bn256():
    # (forced: at 2 images the library takes the 128-column schedule, whose tiles can split)
    return conv_case(256, 512, 14, 1, 1, 2, mode="tf32", tol=1e-2, cfg={"bn": 256, "bk": 32}, expect={"bn": 256})


def fam_tf32_halo():
    return conv_case(128, 128, 14, 3, 1, 2, mode="tf32", tol=1e-2, expect={"halo": 1})


def fam_epix():
    return conv_case(128, 128, 14, 1, 1, 2, scale=True)


def fam_gemm():
    return gemm_case(256, 192, 320)


def fam_gemm_tf32():
    return gemm_case(256, 192, 320, mode="tf32", tol=1e-2)


def fam_gemm_bias():
    return gemm_case(200, 136, 96, bias=True)


def fam_gemm_splitk():
    return gemm_case(128, 128, 2048, cfg={"split_k": 4})


def fam_simt():
    e1 = gemm_case(50, 30, 70, mode="fp32")
    e2 = conv_case(32, 32, 9, 3, 1, 2, mode="fp32")
    e3 = gemm_case(33, 18, 22)  # N % 4 != 0: the tensor-core modes' CUDA-core route
    return max(e1, e2, e3)


def fam_host():
    layer = W.ConvLayer(0, 64, 64, 14, 3, 1)
    x, w, b = W.conv_inputs(layer, 6, seed=2)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    xh = torch.from_numpy(x).pin_memory()
    bd = torch.from_numpy(b).cuda()
    y = P.conv2d_nchw16c_host(xh, pw, bd, stride=1, pad=1, relu=True, chunk=2)
    y2 = P.conv2d_nchw16c_host(xh, pw, bd, stride=1, pad=1, relu=True, chunk=4, x_ready=True)
    torch.cuda.synchronize()
    ref = oracle.conv2d_f64(x, w, b, stride=1, pad=1, relu=True)
    e = max(rel(y.numpy(), ref), rel(y2.numpy(), ref))
    assert e <= 1e-5, e
    return e


def fam_layout():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 19, 9, 11)).astype(np.float32)
    xb = P.ops.to_nchw16c(torch.from_numpy(x).cuda())
    back = P.ops.from_nchw16c(xb, 19)
    w = rng.standard_normal((32, 19, 3, 3)).astype(np.float32)
    wb = P.ops.weights_to_kcrs16c16k(torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), x)
    assert wb.shape == (2, 2, 3, 3, 16, 16)
    return 0.0


def fam_eltwise():
    rng = np.random.default_rng(1)
    y = rng.standard_normal((2, 2, 5, 7, 16)).astype(np.float32)
    y0 = rng.standard_normal(y.shape).astype(np.float32)
    b = rng.standard_normal(32).astype(np.float32)
    yd = torch.from_numpy(y.copy()).cuda()
    P.ops.bias_relu_(yd, torch.from_numpy(b).cuda(), relu=True)
    yd2 = torch.from_numpy(y.copy()).cuda()
    P.ops.accumulate_(yd2, torch.from_numpy(y0).cuda(), torch.from_numpy(b).cuda(), relu=True)
    torch.cuda.synchronize()
    bb = b.reshape(2, 16)[None, :, None, None, :]
    assert np.array_equal(yd.cpu().numpy(), np.maximum(y + bb, 0))
    assert np.array_equal(yd2.cpu().numpy(), np.maximum((y + y0) + bb, 0))
    return 0.0


FAMILIES = {n[4:]: f for n, f in list(globals().items()) if n.startswith("fam_")}


def main(argv):
    names = argv or ["all"]
    if names == ["all"]:
        names = list(FAMILIES)
    assert P.device_ok(), "libpdl.so did not find an sm_100 device"
    for n in names:
        e = FAMILIES[n]()
        print(f"{n}: ok (max-rel {e:.2e}, launches so far {_lib.last_launch_count()})", flush=True)
    print("sanitize_case: all ok")


if __name__ == "__main__":
    main(sys.argv[1:])
