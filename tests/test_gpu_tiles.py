"""Multi-image box tiles.  An M tile is a box of BW x BH output pixels of BNI consecutive
images (one TMA box per 16-channel sub-tile); the library searches (BW, BH, BNI) for the
shape that fills the 128 tensor-core rows best (`pick_box`, csrc/pdl_capi.cu), e.g. 14x1
pixels x 9 images for 28x28 maps instead of 28x4 x 1 (112 rows).  The per-pixel reduction
order does not depend on the tile shape, so every shape must be bitwise equal to the
round-1 single-image geometry (PDL_RASTER_SINGLE_IMAGE_TILES) and within the mode bar of
the fp64 oracle -- for 1x1 / 3x3, stride 1 / 2, halo mode, ragged batches (the last box
holds images past N: TMA zero-fills the loads and clips the stores), explicit boxes
(PDL_RASTER_TILE) and split-K."""
import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import _lib, workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SINGLE = 8  # PDL_RASTER_SINGLE_IMAGE_TILES
BOX = 2     # PDL_RASTER_BOX_TILES (no segment tiles)


def tile(bw, bh, bni):
    return bw << 8 | bh << 16 | bni << 24


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


CASES = [  # (C, K, H, R, stride, N)
    (64, 64, 56, 3, 1, 5),      # layer 3: 8x8 pixels x 2 images, halo mode, odd batch
    (256, 128, 56, 1, 2, 11),   # layer 6: 28x28 out of a stride-2 1x1
    (128, 128, 28, 3, 1, 7),    # layer 7: 14x3 x 3 images, halo mode
    (128, 256, 28, 1, 1, 10),   # layer 8: flattened 1x1, rows of several images
    (256, 256, 14, 3, 1, 7),    # layer 12: 14x3 x 3 images, halo mode
    (256, 128, 14, 1, 1, 19),   # layers 13 / 15
    (256, 128, 14, 1, 2, 37),   # layers 16 / 19: 7x1 pixels x 18 images
    (512, 128, 7, 3, 1, 9),     # layer 17 (whole-image tiles stay)
    (256, 256, 7, 1, 1, 23),    # layers 18 / 20: 25 flattened pixels x 5 images
    (32, 48, 12, 3, 1, 5),      # 12x12, 48 output channels
    (48, 32, 9, 1, 1, 40),      # odd channel-block count (SW64 weights), 9x9 map
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_box_search_equals_single_image_tiles(P, case, mode):
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=31)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=stride, pad=R // 2, relu=True, mode=mode)
    # tf32 with K % 256 == 0 runs 256-column tiles: one segment per tile either way
    new = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": BOX}, **kw)
    old = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": BOX | SINGLE}, **kw)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True)
    assert rel(new.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)
    assert torch.equal(new, old), "the tile shape changed the per-element reduction"
    auto = P.conv2d_nchw16c(xd, pw, bd, **kw)  # default: + segment tiles / split-K when they engage
    assert rel(auto.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)


EXPLICIT = [  # (C, K, H, R, stride, N, (bw, bh, bni))
    (128, 128, 28, 1, 1, 9, (4, 4, 8)),
    (128, 128, 28, 1, 1, 9, (7, 2, 9)),
    (128, 128, 28, 3, 1, 9, (4, 4, 8)),     # 288-pixel halo: over one halo buffer, per-tap boxes
    (128, 128, 28, 3, 1, 9, (7, 4, 4)),     # 216-pixel halo: halo mode
    (256, 128, 28, 1, 2, 20, (14, 1, 9)),
    (64, 64, 56, 3, 1, 3, (16, 8, 1)),
    (64, 64, 56, 3, 1, 3, (56, 1, 2)),
    (512, 128, 7, 3, 1, 20, (7, 1, 18)),    # 7x7 3x3 without the whole-image constraint
    (512, 128, 7, 3, 1, 20, (7, 2, 7)),
    (256, 256, 7, 1, 1, 23, (7, 7, 2)),
]


@pytest.mark.parametrize("case", EXPLICIT, ids=lambda c: "c%dk%dh%dr%ds%dn%d_%dx%dx%d" % (c[:6] + c[6]))
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_explicit_tile_box(P, case, mode):
    C, K, H, R, stride, N, shape = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=33)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=stride, pad=R // 2, relu=True, mode=mode)
    s = _lib.conv_schedule(N, C, K, H, H, R, R, stride, R // 2, _lib.MODES[mode], cfg={"raster": tile(*shape)})
    assert (s["tile_w"], s["tile_h"], s["tile_images"]) == shape and s["seg_rows"] == 0
    got = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": tile(*shape)}, **kw)
    old = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": BOX | SINGLE}, **kw)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True)
    assert rel(got.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)
    assert torch.equal(got, old)
    # the same box with a forced 2-way split of the reduction
    sp = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 2, "raster": tile(*shape), "bn": min(128, s["bn"])}, **kw)
    assert rel(sp.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)
    sp2 = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 2, "raster": tile(*shape), "bn": min(128, s["bn"])}, **kw)
    assert torch.equal(sp, sp2), "split-K result depends on the arrival order"


def _random_cases(n_cases=48, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n_cases:
        R = int(rng.choice([1, 1, 3, 3, 5]))
        S = int(rng.choice([R, R, 1 if R == 1 else 3]))
        stride = int(rng.choice([1, 1, 2]))
        pad_h = int(rng.choice([0, min(R, S) // 2]))
        H, Wd = int(rng.integers(max(R, 2), 41)), int(rng.integers(max(S, 2), 41))
        C = int(rng.choice([16, 32, 48, 64, 128]))
        K = int(rng.choice([16, 32, 64, 128, 256]))
        N = int(rng.integers(1, 41))
        if pad_h >= R or pad_h >= S or H + 2 * pad_h < R or Wd + 2 * pad_h < S:
            continue
        if N * C * H * Wd > 6_000_000 or C * K * R * S > 1_500_000:
            continue
        out.append((C, K, H, Wd, R, S, stride, pad_h, N))
    return out


@pytest.mark.parametrize("case", _random_cases(), ids=lambda c: "c%dk%dh%dw%dr%ds%dst%dp%dn%d" % c)
def test_random_shapes_box_search(P, case):
    """Seeded random shapes (non-square maps and filters, pad 0 or 'same', ragged batches):
    the box search, the round-1 geometry and the fp64 oracle agree -- the first two bitwise."""
    C, K, H, Wd, R, S, stride, pad, N = case
    rng = np.random.default_rng(hash(case) % (1 << 31))
    x = rng.uniform(-1, 1, size=(N, C // 16, H, Wd, 16)).astype(np.float32)
    w = rng.uniform(-1, 1, size=(K // 16, C // 16, R, S, 16, 16)).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, size=(K,)).astype(np.float32)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=stride, pad=pad, relu=True)
    new = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1}, **kw)
    old = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": SINGLE}, **kw)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=pad, relu=True)
    assert rel(new.cpu().numpy(), ref) <= 1e-5
    assert torch.equal(new, old), "the tile shape changed the per-element reduction"
    auto = P.conv2d_nchw16c(xd, pw, bd, **kw)  # + split-K when it engages
    assert rel(auto.cpu().numpy(), ref) <= 1e-5


WIDE3 = [  # (C, K, H, R, stride, N)
    (128, 512, 28, 1, 1, 5),
    (256, 512, 56, 1, 2, 3),
    (512, 1024, 14, 1, 1, 9),
    (64, 256, 12, 3, 1, 4),     # 3x3 with per-tap boxes
    (64, 384, 9, 1, 1, 7),      # K not a multiple of 256: the second N-tile is half empty
    (1024, 256, 7, 1, 1, 37),   # 32 k-blocks = 4 accumulation segments through the single accumulator
]


@pytest.mark.parametrize("case", WIDE3, ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
def test_3xtf32_256_column_tiles(P, case):
    """3xTF32 at 256 columns (one TMEM accumulator drained per segment, setmaxnreg register
    trade): same segments and per-element order as the 128-column tiles, so bitwise equal to
    them, and within 1e-5 of the oracle."""
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=41)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=stride, pad=R // 2, relu=True)
    s = _lib.conv_schedule(N, C, K, H, H, R, R, stride, R // 2, 0, cfg={"bn": 256, "bk": 32})
    assert s["bn"] == 256 and s["resident"] == 0 and s["split"] == 1
    wide = P.conv2d_nchw16c(xd, pw, bd, cfg={"bn": 256, "bk": 32}, **kw)
    narrow = P.conv2d_nchw16c(xd, pw, bd, cfg={"bn": 128, "bk": 32, "split_k": 1}, **kw)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True)
    assert rel(wide.cpu().numpy(), ref) <= 1e-5
    assert torch.equal(wide, narrow)
    assert torch.equal(wide, P.conv2d_nchw16c(xd, pw, bd, cfg={"bn": 256, "bk": 32}, **kw))


def test_3xtf32_256_columns_are_opt_in():
    """Host-only: 256-column 3xTF32 tiles are only taken when asked for (cfg bn=256, bk=32)."""
    for n in (256, 32):
        for l in W.LAYERS:
            assert _lib.conv_schedule(n, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0)["bn"] <= 128
    l = W.LAYERS[18]
    s = _lib.conv_schedule(256, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0, cfg={"bn": 256, "bk": 32})
    assert s["bn"] == 256 and s["n_tiles"] == l.K // 256
