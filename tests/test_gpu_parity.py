"""GPU parity: libpdl.so kernels vs the CPU oracle (bitwise-pinned to the
reference interpreter) on identical seeded inputs.

Tolerance (BASELINE.json north_star): normwise max-relative error
max|y - y_ref| / max|y_ref| <= 1e-5 for 3xTF32 and FP32, <= 1e-2 for TF32.
"""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 1e-2, "fp32": 1e-5}
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def cuda(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------------ golden fixtures
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "conv_*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "fp32"])
def test_conv_vs_reference_golden(P, path, mode):
    g = np.load(path)
    bias = g["bias"] if "bias" in g.files else None
    y = P.conv2d_nchw16c(cuda(g["x"]), cuda(g["w"]), cuda(bias), stride=int(g["stride"]),
                         pad=int(g["pad"]), relu=bool(g["relu"]), mode=mode)
    assert rel(y.cpu().numpy(), g["y"]) <= TOL[mode]


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "gemm_*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "fp32"])
def test_gemm_vs_reference_golden(P, path, mode):
    g = np.load(path)
    c = P.gemm(cuda(g["A"]), cuda(g["B"]), mode=mode)
    assert rel(c.cpu().numpy(), g["C"]) <= TOL[mode]


# ------------------------------------------------------------------ GEMM sweep
_gemm_ref_cache = {}


def _gemm_case(m, n, k, rows):
    key = (m, n, k)
    if key not in _gemm_ref_cache:
        a, b = W.gemm_inputs(m, n, k, seed=7)
        ref = oracle.gemm_f64(a[rows], b)
        _gemm_ref_cache[key] = (a, b, ref)
    return _gemm_ref_cache[key]


@pytest.mark.parametrize("shape", W.GEMM_SWEEP, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "fp32"])
def test_gemm_sweep(P, shape, mode):
    m, n, k = shape
    # rows are independent: for the big shapes check a seeded sample of rows
    rows = np.arange(m) if m <= 1024 else np.sort(
        np.random.default_rng(3).choice(m, 384, replace=False))
    a, b, ref = _gemm_case(m, n, k, rows)
    c = P.gemm(cuda(a), cuda(b), mode=mode).cpu().numpy()
    assert rel(c[rows], ref) <= TOL[mode]


def test_gemm_alpha_beta_relu(P):
    a, b = W.gemm_inputs(200, 136, 72, seed=9)
    c0 = np.random.default_rng(11).uniform(-1, 1, (200, 136)).astype(np.float32)
    ref = oracle.gemm_f64(a, b, c0, alpha=0.5, beta=-2.0)
    c = cuda(c0.copy())
    P.gemm(cuda(a), cuda(b), c, alpha=0.5, beta=-2.0)
    assert rel(c.cpu().numpy(), ref) <= 1e-5
    cr = P.gemm(cuda(a), cuda(b), relu=True).cpu().numpy()
    ref2 = oracle.gemm_f64(a, b)
    assert rel(cr, np.where(0.0 > ref2, 0.0, ref2)) <= 1e-5


# ------------------------------------------------------------------ ResNet-50 layers
_conv_ref_cache = {}


def _conv_ref(layer, n, relu, images=None):
    key = (layer.idx, n, relu, images)
    if key not in _conv_ref_cache:
        x, w, b = W.conv_inputs(layer, n, seed=100 + layer.idx)
        ref = oracle.conv2d_f64(x, w, b if relu else None, stride=layer.stride, pad=layer.pad,
                                relu=relu, images=images)
        _conv_ref_cache[key] = (x, w, b, ref)
    return _conv_ref_cache[key]


@pytest.mark.parametrize("layer", W.LAYERS, ids=lambda l: l.name())
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_resnet_layer_fused(P, layer, mode):
    x, w, b, ref = _conv_ref(layer, 2, True)
    y = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=layer.stride, pad=layer.pad,
                         relu=True, mode=mode, channels=layer.C)
    assert rel(y.cpu().numpy(), ref) <= TOL[mode]


@pytest.mark.parametrize("layer", W.LAYERS, ids=lambda l: l.name())
def test_resnet_layer_unfused_and_prepacked(P, layer):
    x, w, b, ref = _conv_ref(layer, 2, True)
    pw = P.prepack_weights(cuda(w), mode="3xtf32", channels=layer.C)
    y = P.conv2d_nchw16c(cuda(x), pw, None, stride=layer.stride, pad=layer.pad)
    P.bias_relu_(y, cuda(b))
    assert rel(y.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("layer", W.LAYERS, ids=lambda l: l.name())
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_resnet_layer_full_batch_sampled_images(P, layer, mode):
    """BASELINE configs[2]: the full N=28 minibatch (the paper's) of every
    layer on the GPU; the first, a middle and the last image checked against the oracle
    (each image's output depends only on that image)."""
    n = 28
    g = torch.Generator(device="cuda")
    g.manual_seed(500 + layer.idx)
    x = torch.rand((n, layer.C_alloc // 16, layer.H, layer.W, 16), generator=g, device="cuda") * 2 - 1
    if layer.C != layer.C_alloc:
        x[..., layer.C:] = 0
    _, w, b = W.conv_inputs(layer, 1, seed=500 + layer.idx)
    y = P.conv2d_nchw16c(x, cuda(w), cuda(b), stride=layer.stride, pad=layer.pad,
                         relu=True, channels=layer.C, mode=mode)
    for img in (0, 13, n - 1):
        ref = oracle.conv2d_f64(x[img:img + 1].cpu().numpy(), w, b, stride=layer.stride, pad=layer.pad,
                                relu=True)
        assert rel(y[img:img + 1].cpu().numpy(), ref) <= TOL[mode], img


def test_pr1_full(P):
    x, w, _ = W.conv_inputs(W.PR1, 1, seed=1234, bias=False)
    ref = oracle.conv2d_f64(x, w, None, stride=1, pad=1)
    for mode in ("3xtf32", "tf32"):
        y = P.conv2d_nchw16c(cuda(x), cuda(w), None, stride=1, pad=1, mode=mode)
        assert rel(y.cpu().numpy(), ref) <= TOL[mode]


# ------------------------------------------------------------------ properties / edges
def test_deterministic(P):
    layer = W.LAYERS[6]
    x, w, b = W.conv_inputs(layer, 3, seed=1)
    y1 = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=1, pad=1, relu=True)
    y2 = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=1, pad=1, relu=True)
    assert torch.equal(y1, y2)


def test_linearity_in_weights(P):
    """conv(x, w1 + w2) == conv(x, w1) + conv(x, w2) within 3xTF32 tolerance."""
    layer = W.LAYERS[11]
    x, w1, _ = W.conv_inputs(layer, 2, seed=2)
    _, w2, _ = W.conv_inputs(layer, 2, seed=5)
    ya = P.conv2d_nchw16c(cuda(x), cuda(w1 + w2), stride=1, pad=1).cpu().numpy()
    yb = (P.conv2d_nchw16c(cuda(x), cuda(w1), stride=1, pad=1)
          + P.conv2d_nchw16c(cuda(x), cuda(w2), stride=1, pad=1)).cpu().numpy()
    assert rel(ya, yb.astype(np.float64)) <= 2e-5


def test_batch_shard_concat_equals_full(P):
    """The batch-sharding rule: per-shard outputs concatenate to the full output."""
    layer = W.LAYERS[2]
    x, w, b = W.conv_inputs(layer, 4, seed=8)
    full = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=1, pad=1, relu=True)
    parts = [P.conv2d_nchw16c(cuda(x[i:i + 2]), cuda(w), cuda(b), stride=1, pad=1, relu=True)
             for i in (0, 2)]
    assert torch.equal(full, torch.cat(parts))


@pytest.mark.parametrize("h,r,stride", [(1, 1, 1), (3, 3, 1), (5, 3, 2), (9, 1, 2), (130, 1, 1),
                                        (17, 3, 1), (8, 7, 2)])
def test_ragged_spatial(P, h, r, stride):
    layer = W.ConvLayer(99, 32, 48, h, r, stride)
    if layer.P <= 0:
        pytest.skip("empty output")
    x, w, b = W.conv_inputs(layer, 3, seed=h)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=layer.pad, relu=True)
    y = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=stride, pad=layer.pad, relu=True)
    assert rel(y.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("c,r,stride,h", [(3, 7, 2, 30), (4, 3, 1, 9), (1, 5, 2, 11), (3, 7, 2, 224)])
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "fp32"])
def test_narrow_channel_stem(P, c, r, stride, h, mode):
    """C <= 4 real channels in one padded 16-block: the stem kernel must ignore
    the padding channels even if they hold garbage."""
    layer = W.ConvLayer(98, c, 64 if h != 224 else 128, h, r, stride)
    n = 2 if h < 224 else 1
    x, w, b = W.conv_inputs(layer, n, seed=c * 100 + r)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=layer.pad, relu=True)
    xg = x.copy()
    xg[..., c:] = 7.0  # garbage in the padding channels must not leak in
    wg = w.copy()
    wg[:, :, :, :, c:, :] = -3.0
    y = P.conv2d_nchw16c(cuda(xg), cuda(wg), cuda(b), stride=stride, pad=layer.pad, relu=True,
                         mode=mode, channels=c)
    assert rel(y.cpu().numpy(), ref) <= TOL[mode]


@pytest.mark.parametrize("cluster", [1, 2, 4])
@pytest.mark.parametrize("layer", [l for l in W.LAYERS if l.idx in (3, 6, 7, 13, 17)],
                         ids=lambda l: l.name())
def test_cluster_multicast_conv(P, layer, cluster):
    """Weight tiles multicast across clusters of 1/2/4 CTAs give identical results
    (same reduction order per element) and match the oracle."""
    x, w, b, ref = _conv_ref(layer, 2, True)
    ys = []
    for mode in ("3xtf32", "tf32"):
        y = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=layer.stride, pad=layer.pad,
                             relu=True, mode=mode, cfg={"cluster_m": cluster, "split_k": 1})
        assert rel(y.cpu().numpy(), ref) <= TOL[mode]
        ys.append(y)
    y1 = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), stride=layer.stride, pad=layer.pad,
                          relu=True, cfg={"cluster_m": 1, "split_k": 1})
    assert torch.equal(ys[0], y1)


@pytest.mark.parametrize("cluster", [1, 2, 4])
@pytest.mark.parametrize("shape", [(300, 192, 100), (1024, 1024, 1024), (49, 2048, 512)],
                         ids=lambda s: "x".join(map(str, s)))
def test_cluster_multicast_gemm(P, shape, cluster):
    m, n, k = shape
    a, b = W.gemm_inputs(m, n, k, seed=17)
    ref = oracle.gemm_f64(a, b)
    for mode in ("3xtf32", "tf32"):
        c = P.gemm(cuda(a), cuda(b), mode=mode, cfg={"cluster_m": cluster}).cpu().numpy()
        assert rel(c, ref) <= TOL[mode]


def test_bad_shapes_raise(P):
    x = torch.zeros((1, 1, 4, 4, 16), device="cuda")
    w = torch.zeros((1, 1, 3, 3, 16, 16), device="cuda")
    with pytest.raises(P.PdlShapeError):
        P.conv2d_nchw16c(x, w, stride=3, pad=1)
    with pytest.raises(ValueError):
        P.conv2d_nchw16c(x, w, mode="int8")
    with pytest.raises(ValueError):
        P.conv2d_nchw16c(torch.zeros((1, 2, 4, 4, 16), device="cuda"), w)


@pytest.mark.parametrize("shape", [(3, 64, 256, 7, 1, 1), (2, 96, 512, 9, 1, 1), (1, 256, 768, 14, 2, 1),
                                   (5, 512, 256, 5, 1, 1), (2, 32, 1024, 28, 2, 1), (2, 16, 256, 9, 1, 3),
                                   (3, 64, 512, 7, 1, 3), (2, 32, 256, 15, 2, 3), (1, 32, 256, 12, 1, 5)])
def test_tf32_wide_tiles(P, shape):
    """TF32 convs with K % 256 == 0 default to 256-column tiles (streaming epilogue);
    ragged pixel tails, strides, filter sizes and channel counts against the oracle and
    the 128-column tiles (bitwise while C*R*S <= 256 keeps both in one accumulation
    segment)."""
    n, C, K, H, stride, R = shape
    pad = R // 2
    rng = np.random.default_rng(sum(shape))
    x = (rng.random((n, C // 16, H, H, 16), np.float32) * 2 - 1).astype(np.float32)
    w = ((rng.random((K // 16, C // 16, R, R, 16, 16)) * 2 - 1) / np.sqrt(C * R * R)).astype(np.float32)
    b = rng.random(K, np.float32)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=pad, relu=True)
    kw = dict(stride=stride, pad=pad, relu=True, mode="tf32")
    wide = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), **kw)
    assert rel(wide.cpu().numpy(), ref) <= TOL["tf32"]
    narrow = P.conv2d_nchw16c(cuda(x), cuda(w), cuda(b), cfg={"bn": 128, "bk": 32 if C % 32 == 0 else 16, "split_k": 1}, **kw)
    if C * R * R <= 256:
        assert torch.equal(wide, narrow)
    else:
        assert rel(wide.cpu().numpy(), narrow.cpu().numpy().astype(np.float64)) <= 1e-5
