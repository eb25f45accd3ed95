"""Compact narrow-channel input (PDL_X_NCHW4C): x as [N][H][W][4] instead of
nChw16c's 64-byte pixels (the stem's padded-input traffic).
Same kernel, same arithmetic order: the result must be BITWISE equal to the
nChw16c call, and within the mode bar of the fp64 oracle."""
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


CASES = [  # (C, K, H, R, stride, N)
    (3, 64, 224, 7, 2, 2),   # ResNet-50 stem (packed reduction, even/odd column boxes)
    (3, 64, 37, 7, 2, 3),    # odd size: clipped tiles
    (3, 32, 30, 7, 1, 2),    # stride 1 (one dense halo box)
    (4, 64, 28, 5, 2, 2),    # row-form reduction, 4 real channels
    (1, 16, 19, 3, 1, 2),    # one channel
    (2, 48, 24, 3, 2, 1),
]


@pytest.mark.parametrize("mode,tol", [("3xtf32", 1e-5), ("tf32", 1e-2)])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
def test_compact_equals_nchw16c_and_oracle(P, case, mode, tol):
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=21)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode, channels=C)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    x4 = xd[:, 0, :, :, :4].contiguous()
    assert x4.shape == (N, H, H, 4)
    y16 = P.conv2d_nchw16c(xd, pw, bd, stride=stride, pad=R // 2, relu=True, mode=mode, channels=C)
    y4 = P.conv2d_nchw16c(x4, pw, bd, stride=stride, pad=R // 2, relu=True, mode=mode, channels=C)
    assert torch.equal(y4, y16)
    ref = oracle.conv2d_f64(x, w, b, stride=stride, pad=R // 2, relu=True)
    assert rel(y4.cpu().numpy(), ref) <= tol


def test_pack_nchw4c_and_raw_weight_call(P):
    rng = np.random.default_rng(5)
    xn = rng.uniform(-1, 1, (3, 3, 33, 29)).astype(np.float32)
    x4 = P.to_nchw4c(torch.from_numpy(xn).cuda())
    want = np.zeros((3, 33, 29, 4), np.float32)
    want[..., :3] = xn.transpose(0, 2, 3, 1)
    assert np.array_equal(x4.cpu().numpy(), want)
    x16 = P.to_nchw16c(torch.from_numpy(xn).cuda())
    wn = rng.uniform(-1, 1, (32, 3, 7, 7)).astype(np.float32)
    wb = P.weights_to_kcrs16c16k(torch.from_numpy(wn).cuda())
    y4 = P.conv2d_nchw16c(x4, wb, None, stride=2, pad=3, channels=3)      # raw weights
    y16 = P.conv2d_nchw16c(x16, wb, None, stride=2, pad=3, channels=3)
    assert torch.equal(y4, y16)


def test_compact_host_pipeline(P):
    layer = W.ConvLayer(0, 3, 64, 64, 7, 2)
    x, w, b = W.conv_inputs(layer, 10, seed=8)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), channels=3)
    bd = torch.from_numpy(b).cuda()
    x4h = torch.from_numpy(np.ascontiguousarray(x[:, 0, :, :, :4])).pin_memory()
    y_dev = P.conv2d_nchw16c(x4h.cuda(), pw, bd, stride=2, pad=3, relu=True, channels=3)
    for chunk in (0, 1, 3, 10):
        y = P.conv2d_nchw16c_host(x4h, pw, bd, stride=2, pad=3, relu=True, chunk=chunk)
        torch.cuda.synchronize()
        assert torch.equal(y, y_dev.cpu()), f"chunk={chunk}"
    ref = oracle.conv2d_f64(x, w, b, stride=2, pad=3, relu=True)
    assert rel(y.numpy(), ref) <= 1e-5


def test_compact_rejected_off_the_narrow_path(P):
    from paper_2006_02230_b200._lib import PdlShapeError
    layer = W.ConvLayer(0, 64, 64, 14, 3, 1)
    x, w, b = W.conv_inputs(layer, 1, seed=1)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    x4 = torch.zeros((1, 14, 14, 4), device="cuda")
    with pytest.raises(ValueError):
        P.conv2d_nchw16c(x4, pw, None, stride=1, pad=1)
    layer = W.ConvLayer(0, 3, 16, 12, 3, 1)
    x, w, b = W.conv_inputs(layer, 1, seed=1)
    with pytest.raises(PdlShapeError):   # exact-fp32 CUDA-core conv reads nChw16c
        P.conv2d_nchw16c(torch.zeros((1, 12, 12, 4), device="cuda"), torch.from_numpy(w).cuda(), None,
                         stride=1, pad=1, mode="fp32", channels=3)
