"""Halo mode (3xTF32, stride-1 spatial convs): the input halo of a tile is loaded
once per channel group and the staging warps read each tap's shifted window from
shared memory, instead of one TMA box per tap.  Same MMAs in the same order, so
results are bitwise equal to per-tap boxes; checked against the fp64 oracle too,
with split-K ranges that start in the middle of a channel group."""
import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NO_HALO = 16  # PDL_RASTER_NO_HALO


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


CASES = [  # (C, K, H, R, N): ResNet 3x3 shapes and odd ones
    (64, 64, 56, 3, 2),      # layer 3 (BN=64, 64-channel k-blocks: stays on per-tap boxes)
    (128, 128, 28, 3, 2),    # layer 7
    (256, 256, 14, 3, 3),    # layer 12
    (512, 512, 7, 3, 3),     # layer 17 (two images per tile)
    (48, 32, 9, 3, 3),       # 16-channel k-blocks (CG = 1), ragged map
    (32, 64, 20, 5, 2),      # 5x5 filter
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%dk%dh%dr%dn%d" % c)
@pytest.mark.parametrize("split", [1, 3])
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_halo_bitwise_equals_per_tap_boxes(P, case, split, mode):
    """TF32 halo convs stage A through TMEM (TS MMAs) while per-tap TF32 convs read A
    from shared memory (SS MMAs): the tensor core truncates the same fp32 bits either
    way, so they agree bitwise too."""
    C, K, H, R, N = case
    layer = W.ConvLayer(0, C, K, H, R, 1)
    x, w, b = W.conv_inputs(layer, N, seed=31)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    kw = dict(stride=1, pad=R // 2, relu=True, mode=mode)
    halo = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": split, "cluster_m": 1}, **kw)
    taps = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": split, "cluster_m": 1, "raster": NO_HALO}, **kw)
    assert torch.equal(halo, taps)
    ref = oracle.conv2d_f64(x, w, b, stride=1, pad=R // 2, relu=True)
    assert rel(halo.cpu().numpy(), ref) <= (1e-5 if mode == "3xtf32" else 1e-2)


def test_halo_single_buffer_64_channel_kblocks(P):
    """PDL_RASTER_HALO_CG4: 3xTF32 halo with 64-channel k-blocks and one halo buffer."""
    for case in [(64, 64, 56, 3, 2), (128, 64, 14, 3, 3)]:
        C, K, H, R, N = case
        layer = W.ConvLayer(0, C, K, H, R, 1)
        x, w, b = W.conv_inputs(layer, N, seed=41)
        pw = P.prepack_weights(torch.from_numpy(w).cuda())
        xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
        kw = dict(stride=1, pad=R // 2, relu=True)
        a = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": NO_HALO}, **kw)
        c = P.conv2d_nchw16c(xd, pw, bd, cfg={"split_k": 1, "raster": 64}, **kw)
        assert torch.equal(a, c)
