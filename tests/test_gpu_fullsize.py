"""BASELINE full sizes: every ResNet-50 layer at the 256-image minibatch of the
scaling config (configs[4]), in 3xTF32 and TF32, checked on sampled images
against the fp64 oracle (each image's output depends only on that image), and
the 8-GPU shard (the last 32 images run as their own batch, the way rank 7 of
8 runs them) against the same images of the full run."""
import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 1e-2}
N = 256


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


@pytest.mark.parametrize("layer", W.LAYERS, ids=lambda l: l.name())
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_full_minibatch_sampled_images_and_shard(P, layer, mode):
    g = torch.Generator(device="cuda")
    g.manual_seed(7000 + layer.idx)
    x = torch.rand((N, layer.C_alloc // 16, layer.H, layer.W, 16), generator=g, device="cuda") * 2 - 1
    if layer.C != layer.C_alloc:
        x[..., layer.C:] = 0
    _, w, b = W.conv_inputs(layer, 1, seed=layer.idx)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode, channels=layer.C)
    bd = torch.from_numpy(b).cuda()
    kw = dict(stride=layer.stride, pad=layer.pad, relu=True, mode=mode)
    y = P.conv2d_nchw16c(x, pw, bd, **kw)
    for img in (0, 131, N - 1):
        xi = x[img:img + 1].cpu().numpy()
        ref = oracle.conv2d_f64(xi, w, b, stride=layer.stride, pad=layer.pad, relu=True)
        assert rel(y[img:img + 1].cpu().numpy(), ref) <= TOL[mode], img
    shard = P.conv2d_nchw16c(x[N - 32:].contiguous(), pw, bd, **kw)
    full = y[N - 32:].cpu().numpy().astype(np.float64)
    assert rel(shard.cpu().numpy(), full) <= (2e-6 if mode == "3xtf32" else 1e-3)
