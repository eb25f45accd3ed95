"""Split-K (the small-batch schedule): each tile's reduction is cut into ranges
computed by different CTAs; the last CTA of a tile sums the partials in range
order and runs the fused epilogue.  Checked against the fp64 oracle (1e-5,
3xTF32), for determinism (two launches bitwise equal, whatever the arrival
order), and for the self-resetting tile counters (many launches in a row)."""
import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


CONV = [  # (C, K, H, R, stride, N): ResNet-50 layers at small batches + odd shapes
    (512, 512, 7, 3, 1, 2),     # layer 17
    (1024, 512, 14, 1, 2, 2),   # layer 16
    (2048, 512, 7, 1, 1, 1),    # layer 20
    (256, 256, 14, 3, 1, 1),    # layer 12
    (48, 32, 9, 3, 2, 3),       # odd channel blocks (CG = 1)
]


@pytest.mark.parametrize("case", CONV, ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
@pytest.mark.parametrize("split", [0, 2, 3, 7])
def test_conv_splitk_vs_oracle(P, case, split):
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=5)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    cfg = {"split_k": split}
    y1 = P.conv2d_nchw16c(xd, pw, bd, stride=stride, pad=R // 2, relu=True, cfg=cfg)
    y2 = P.conv2d_nchw16c(xd, pw, bd, stride=stride, pad=R // 2, relu=True, cfg=cfg)
    assert torch.equal(y1, y2), "split-K result depends on CTA arrival order"
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True)
    assert rel(y1.cpu().numpy(), ref) <= 1e-5


def test_conv_auto_split_engages_and_matches_unsplit(P):
    from paper_2006_02230_b200 import _lib
    L = _lib.lib()
    assert L.pdl_conv2d_splitk_workspace_bytes(2, 512, 512, 7, 7, 3, 3, 1, 1, 0, None) > 0
    layer = W.ConvLayer(0, 512, 512, 7, 3, 1)
    x, w, b = W.conv_inputs(layer, 2, seed=9)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    auto = P.conv2d_nchw16c(xd, pw, bd, stride=1, pad=1, relu=True)
    off = P.conv2d_nchw16c(xd, pw, bd, stride=1, pad=1, relu=True, cfg={"split_k": 1})
    ref = oracle.conv2d_f64(x, w, b, stride=1, pad=1, relu=True)
    assert rel(auto.cpu().numpy(), ref) <= 1e-5 and rel(off.cpu().numpy(), ref) <= 1e-5
    # both schedules are fp32-accurate; they differ only by re-association
    assert rel(auto.cpu().numpy(), off.cpu().numpy().astype(np.float64)) <= 1e-5


def test_counters_reset_across_many_launches(P):
    layer = W.ConvLayer(0, 256, 256, 14, 3, 1)
    x, w, b = W.conv_inputs(layer, 1, seed=3)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    first = P.conv2d_nchw16c(xd, pw, bd, stride=1, pad=1, relu=True, cfg={"split_k": 4})
    y = torch.empty_like(first)
    for _ in range(50):
        P.conv2d_nchw16c(xd, pw, bd, stride=1, pad=1, relu=True, cfg={"split_k": 4}, out=y)
    assert torch.equal(first, y)


def test_raw_weight_call_with_split(P):
    layer = W.ConvLayer(0, 512, 512, 7, 3, 1)
    x, w, b = W.conv_inputs(layer, 1, seed=4)
    y = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(),
                         torch.from_numpy(b).cuda(), stride=1, pad=1, relu=True)
    ref = oracle.conv2d_f64(x, w, b, stride=1, pad=1, relu=True)
    assert rel(y.cpu().numpy(), ref) <= 1e-5


def test_workspace_shared_across_shapes(P):
    """One cached workspace serves split plans of different tile counts in a row:
    the counters sit in a fixed block, so one plan's partials never become another
    plan's counters (regression: a 64-column-tile plan after a 128-column one)."""
    for (m, n, k, bn) in [(1024, 1024, 1024, 128), (1024, 1024, 1024, 64), (512, 512, 4096, 128),
                          (1024, 1024, 1024, 64), (256, 192, 2048, 64)]:
        a, bm = W.gemm_inputs(m, n, k, seed=m + bn)
        for sk in (2, 3):
            c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(),
                       cfg={"split_k": sk, "bn": bn})
            assert rel(c.cpu().numpy(), oracle.gemm_f64(a, bm)) <= 1e-5, (m, n, k, bn, sk)


@pytest.mark.parametrize("mnk", [(1024, 1024, 1024), (512, 512, 512), (256, 192, 2048),
                                 (100, 68, 3000)])
@pytest.mark.parametrize("split", [0, 3])
def test_gemm_splitk_vs_oracle(P, mnk, split):
    m, n, k = mnk
    a, bm = W.gemm_inputs(m, n, k, seed=2)
    c0 = np.random.default_rng(7).uniform(-1, 1, size=(m, n)).astype(np.float32)
    c = torch.from_numpy(c0).cuda()
    P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(), c, alpha=0.5, beta=-2.0,
           cfg={"split_k": split})
    ref = 0.5 * oracle.gemm_f64(a, bm) - 2.0 * c0.astype(np.float64)
    assert rel(c.cpu().numpy(), ref) <= 1e-5


# Halo mode + short split-K ranges, repeated: the staging warps' generic-proxy reads of a
# halo buffer must be fenced (fence.proxy.async) before the buffer is released to the
# next TMA write.  Without the fence a 1-k-block range re-loaded the buffer while a warp
# still read the last tap (wrong rows in ~1 of 4 launches).  Every repetition must be
# bitwise equal to the first and within the mode's bar of the unsplit schedule.
RACE = [  # (C, K, H, R, N, mode, extra cfg, splits)
    (64, 64, 56, 3, 1, "3xtf32", {"bk": 32}, (18, 19, 24)),    # PR1, 1-k-block ranges
    (64, 64, 56, 3, 1, "tf32", {"bk": 32}, (18, 19)),
    (512, 512, 7, 3, 32, "tf32", {}, (3, 4, 6, 9)),             # layer 17, 8-image shard
    (512, 512, 7, 3, 32, "3xtf32", {}, (9, 12, 18)),
    (256, 256, 14, 3, 8, "3xtf32", {}, (15, 16, 21)),           # layer 12
    (64, 64, 56, 3, 2, "3xtf32", {}, (13, 18)),                 # layer 3
]


@pytest.mark.parametrize("case", RACE, ids=lambda c: "c%dk%dh%dr%dn%d_%s" % c[:6])
def test_halo_splitk_repeated_launches_are_identical(P, case):
    C, K, H, R, N, mode, extra, splits = case
    layer = W.ConvLayer(0, C, K, H, R, 1)
    g = torch.Generator(device="cuda")
    g.manual_seed(C + K + N)
    x = torch.rand((N, C // 16, H, H, 16), generator=g, device="cuda") * 2 - 1
    w = torch.rand((K // 16, C // 16, R, R, 16, 16), generator=g, device="cuda") * 2 - 1
    pw = P.prepack_weights(w, mode=mode)
    base = P.conv2d_nchw16c(x, pw, stride=1, pad=R // 2, mode=mode, cfg=dict(extra, split_k=1))
    scale = float(base.abs().max())
    tol = 1e-5 if mode == "3xtf32" else 1e-3
    for s in splits:
        cfg = dict(extra, split_k=s)
        first = P.conv2d_nchw16c(x, pw, stride=1, pad=R // 2, mode=mode, cfg=cfg)
        assert float((first - base).abs().max()) <= tol * scale, (s, "vs unsplit")
        out = torch.empty_like(first)
        for rep in range(6):
            P.conv2d_nchw16c(x, pw, stride=1, pad=R // 2, mode=mode, cfg=cfg, out=out)
            assert torch.equal(out, first), (s, rep)
