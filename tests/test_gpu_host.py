"""Host-buffer convolution (pdl_conv2d_fwd_host): the reference's interpret()
contract -- host arrays in, host arrays out (simcache.py:89-204, inputs copied
at :110) -- with image chunks pipelined over three streams.  Every chunking
must be BITWISE equal to the device-resident call on the same inputs (the
kernels are batch-position independent), and within 1e-5 of the fp64 oracle."""
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


CASES = [  # (C, K, H, R, stride, N)
    (3, 64, 40, 7, 2, 5),     # stem kernel
    (64, 64, 14, 3, 1, 7),    # 3x3
    (256, 128, 14, 1, 2, 4),  # 1x1 stride 2
    (64, 256, 9, 1, 1, 3),    # 1x1 flattened, resident weights
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%dk%dh%dr%ds%dn%d" % c)
@pytest.mark.parametrize("chunk", [0, 1, 2, 64])
def test_host_pipeline_bitwise_equals_device(P, case, chunk):
    C, K, H, R, stride, N = case
    layer = W.ConvLayer(0, C, K, H, R, stride)
    x, w, b = W.conv_inputs(layer, N, seed=11)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), channels=C)
    bd = torch.from_numpy(b).cuda()
    # the host pipeline runs unsplit chunks (PCIe-bound; no split-K workspace), so the
    # device reference is the unsplit schedule too
    y_dev = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), pw, bd, stride=stride, pad=R // 2,
                             relu=True, cfg={"split_k": 1}).cpu()
    xh = torch.from_numpy(x).pin_memory()
    y_host = P.conv2d_nchw16c_host(xh, pw, bd, stride=stride, pad=R // 2, relu=True, chunk=chunk)
    torch.cuda.current_stream().synchronize()
    assert not y_host.is_cuda
    assert torch.equal(y_host, y_dev)


def test_host_pipeline_vs_oracle_and_reuse(P):
    """Two back-to-back calls reuse the staging slots; both must be correct."""
    layer = W.ConvLayer(0, 32, 48, 12, 3, 1)
    outs, refs = [], []
    for seed in (1, 2):
        x, w, b = W.conv_inputs(layer, 6, seed=seed)
        pw = P.prepack_weights(torch.from_numpy(w).cuda())
        outs.append(P.conv2d_nchw16c_host(torch.from_numpy(x).pin_memory(), pw,
                                          torch.from_numpy(b).cuda(), stride=1, pad=1, relu=True,
                                          chunk=1))
        refs.append(oracle.conv2d_f64(x, w, b, stride=1, pad=1, relu=True))
    torch.cuda.synchronize()
    for y, ref in zip(outs, refs):
        err = float(np.abs(y.numpy() - ref).max() / np.abs(ref).max())
        assert err <= 1e-5


def test_host_pipeline_rejects_bad_arguments(P):
    layer = W.ConvLayer(0, 16, 16, 8, 3, 1)
    x, w, b = W.conv_inputs(layer, 2, seed=0)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    with pytest.raises(TypeError):
        P.conv2d_nchw16c_host(torch.from_numpy(x).cuda(), pw, None, pad=1)
    with pytest.raises(TypeError):
        P.conv2d_nchw16c_host(torch.from_numpy(x), torch.from_numpy(w).cuda(), None, pad=1)
    with pytest.raises(ValueError):
        P.conv2d_nchw16c_host(torch.from_numpy(x), pw, None, pad=1,
                              out=torch.empty((2, 1, 8, 7, 16)))
    with pytest.raises(P.PdlError):
        P.conv2d_nchw16c_host(torch.from_numpy(x), pw, None, pad=1, chunk=-1)
