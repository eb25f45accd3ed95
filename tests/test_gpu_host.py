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


def test_host_calls_overlap_across_layers(P):
    """x_ready=True: consecutive calls with different layer shapes share the staging
    workspace while an earlier call's copies out may still run; every output must
    equal the device call (x and y halves of the workspace never alias)."""
    layers = [W.ConvLayer(0, 64, 128, 14, 3, 1), W.ConvLayer(0, 128, 64, 28, 1, 2),
              W.ConvLayer(0, 3, 64, 40, 7, 2), W.ConvLayer(0, 64, 256, 9, 1, 1)]
    outs, refs = [], []
    for i, layer in enumerate(layers):
        x, w, b = W.conv_inputs(layer, 6, seed=30 + i)
        pw = P.prepack_weights(torch.from_numpy(w).cuda(), channels=layer.C)
        bd = torch.from_numpy(b).cuda()
        refs.append(P.conv2d_nchw16c(torch.from_numpy(x).cuda(), pw, bd, stride=layer.stride,
                                     pad=layer.pad, relu=True, cfg={"split_k": 1}).cpu())
        outs.append((torch.from_numpy(x).pin_memory(), pw, bd, layer))
    torch.cuda.synchronize()
    ys = [P.conv2d_nchw16c_host(xh, pw, bd, stride=l.stride, pad=l.pad, relu=True, chunk=2,
                                x_ready=True) for xh, pw, bd, l in outs * 2]
    torch.cuda.synchronize()
    for i, y in enumerate(ys):
        assert torch.equal(y, refs[i % len(refs)])


def test_host_chained_layers_keep_stream_order(P):
    """Without x_ready, a call whose x_host is the previous call's y_host waits for
    those copies out (the reference's chained nests)."""
    l1 = W.ConvLayer(0, 32, 32, 12, 3, 1)
    x, w1, b1 = W.conv_inputs(l1, 4, seed=40)
    _, w2, b2 = W.conv_inputs(l1, 4, seed=41)
    pw1 = P.prepack_weights(torch.from_numpy(w1).cuda())
    pw2 = P.prepack_weights(torch.from_numpy(w2).cuda())
    bd1, bd2 = torch.from_numpy(b1).cuda(), torch.from_numpy(b2).cuda()
    y1 = P.conv2d_nchw16c_host(torch.from_numpy(x).pin_memory(), pw1, bd1, pad=1, relu=True, chunk=1)
    y2 = P.conv2d_nchw16c_host(y1, pw2, bd2, pad=1, relu=True, chunk=1)
    torch.cuda.synchronize()
    d1 = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), pw1, bd1, pad=1, relu=True, cfg={"split_k": 1})
    d2 = P.conv2d_nchw16c(d1, pw2, bd2, pad=1, relu=True, cfg={"split_k": 1})
    assert torch.equal(y2, d2.cpu())
