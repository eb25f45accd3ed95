"""Segment tiles: for small output maps (14x14, 7x7) an M tile is the next T
"bands" of the (image group, output row) sequence -- a band is one output row of
one image (even Q) or of two images (odd Q) -- loaded as up to three exact-height
boxes stacked at 128-byte-aligned smem offsets, so tiles span images and fill
126 of 128 rows instead of 98 on average.  The TMA swizzle follows absolute shared-memory address bits
(scripts/tma_swizzle_probe.cu), so the stack is the canonical SW64 tile.  Checked
against the fp64 oracle and bitwise against box tiles (same per-element reduction
order), for stride 1 / 2, 1x1 / 3x3, odd batches, TF32 and split-K."""
import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BOX = 2  # PDL_RASTER_BOX_TILES
SEG = 4  # PDL_RASTER_SEG_TILES (also when they do not remove a wave)


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


CASES = [  # (C, K, H, R, stride, N)
    (256, 256, 14, 3, 1, 3),    # 14x14 3x3 (layer 12 shape), one row per segment
    (256, 128, 14, 1, 1, 5),    # 14x14 1x1 (layer 13/15 shape, otherwise flattened)
    (512, 256, 28, 1, 2, 3),    # 28 -> 14 stride 2 (layer 11 / 14 shape)
    (512, 128, 7, 3, 1, 9),     # 7x7 3x3 (layer 17 shape): two-image bands, odd N
    (256, 256, 7, 1, 1, 10),    # 7x7 1x1 (layer 18 / 20 shape): up to three boxes per tile
    (256, 128, 14, 1, 2, 9),    # 14 -> 7 stride 2 (layer 16 / 19 shape)
    (64, 32, 16, 3, 1, 3),      # 16x16: 8 rows per tile, whole tiles inside images
    (32, 48, 12, 3, 1, 5),      # 12x12: 10 rows per tile (the most row counts)
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_segment_tiles(P, case, mode):
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=21)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=stride, pad=R // 2, relu=True, mode=mode)
    seg = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": SEG}, **kw)
    box = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": BOX}, **kw)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True)
    assert rel(seg.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)
    assert torch.equal(seg, box), "segment tiles changed the per-element reduction"
    auto = P.conv2d_nchw16c(xd, pw, bd, **kw)  # + split-K when it engages
    assert rel(auto.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)


def test_resnet_small_map_layers_full_batch_sample(P):
    """The ResNet-50 14x14 / 7x7 layers at 33 images (odd, > one wave of tiles)."""
    for layer in [l for l in W.LAYERS if l.P in (7, 14)]:
        x, w, b = W.conv_inputs(layer, 33, seed=layer.idx)
        pw = P.prepack_weights(torch.from_numpy(w).cuda())
        y = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), pw, torch.from_numpy(b).cuda(),
                             stride=layer.stride, pad=layer.pad, relu=True)
        yn = y.cpu().numpy()
        for i in (0, 16, 32):  # sampled images vs the oracle (the full batch is slow on CPU)
            ref = oracle.conv2d_f64(x[i:i + 1], w, b, stride=layer.stride, pad=layer.pad, relu=True)
            assert rel(yn[i:i + 1], ref) <= 1e-5, layer.name()


@pytest.mark.parametrize("case", [(64, 256, 56, 1, 1, 2), (128, 128, 28, 3, 1, 3), (256, 128, 28, 1, 2, 2),
                                  (512, 512, 7, 3, 1, 3), (48, 32, 9, 3, 2, 3), (3, 64, 40, 7, 2, 2),
                                  (256, 1024, 14, 1, 1, 4)],
                         ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
@pytest.mark.parametrize("split", [1, 3])
def test_m_fastest_tile_order_bitwise(P, case, split):
    """PDL_RASTER_M_FASTEST (raster bit 0, the tile-loop interchange of the variant
    space): output-pixel tiles fastest instead of output-channel tiles.  Every tile
    reduces in the same order, so results are bitwise equal (segment, box and
    split-K tiles; silently ignored where CTAs pin an N-tile: stem, resident weights)."""
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=23)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), channels=C)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=stride, pad=R // 2, relu=True)
    n_first = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": split}, **kw)
    sentinel = torch.full_like(n_first, float("nan"))
    m_first = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": split, "raster": 1}, out=sentinel, **kw)
    assert torch.equal(n_first, m_first)
