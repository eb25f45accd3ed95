"""Alg. 3 on the GPU: the fused epilogues (ReLU6, batch-norm inference scale +
shift, bias + ReLU) in the tile kernels, the stand-alone element-wise kernel, and
fusion.FusedNest / two-operator programs through the executor, against the
reference's own execution of the same programs (tests/golden/fusion_ref.json)
and the float64 oracle."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import interp
from paper_2006_02230_b200 import fusion as F
from paper_2006_02230_b200 import loopnest as L
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF = json.load(open(os.path.join(GOLD, "fusion_ref.json")))
TOL = {"3xtf32": 1e-5, "tf32": 1e-2}


def rel(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30))


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def epi_ref(y, bias=None, scale=None, act=None):
    """float64 epilogue in the reference's order: scale, shift, then max / min."""
    y = np.array(y, np.float64)
    sh = (1, -1, 1, 1, 16)
    if scale is not None:
        y = y * np.asarray(scale, np.float64).reshape(sh)
    if bias is not None:
        y = y + np.asarray(bias, np.float64).reshape(sh)
    if act in ("relu", "relu6"):
        y = np.where(0.0 > y, 0.0, y)
    if act == "relu6":
        y = np.where(6.0 < y, 6.0, y)
    return y


@pytest.mark.parametrize("case", [c for c in sorted(REF) if not REF[c]["ew_first"]])
@pytest.mark.parametrize("form", ["fused_nest", "program"])
def test_executor_matches_reference_execution(P, case, form):
    g = REF[case]
    prog = L.parse_program(g["text"])
    if form == "fused_nest":
        nests = F.fuse(F.OperatorPair(prog.nests[0], prog.nests[1]), g["binding"])
    else:
        nests = prog
    inputs = {k: np.array(v) for k, v in g["inputs"].items()}
    got = P.execute(nests, g["binding"], inputs)
    # normwise against the pre-activation scale (ReLU6 saturates the output at 6, far
    # below the accumulated values): max|heavy output| times the largest per-channel
    # factor the element-wise statement applies
    pre = interp.interpret(prog.nests[0], g["binding"], inputs)
    ew = prog.nests[1].statements()[0]
    factor = max([1.0] + [float(np.abs(inputs[a.array]).max()) for a in
                          L.expr_accesses(ew.expr) if a.array != ew.target.array])
    for arr, ref in g["fused"].items():
        denom = max(float(np.abs(pre[arr]).max()) * factor, float(np.abs(ref).max()), 1e-30)
        assert float(np.abs(got[arr] - np.array(ref)).max()) / denom <= TOL["3xtf32"], arr


def test_element_wise_first_on_gemm_output_is_refused(P):
    g = REF["relu_then_gemm"]
    prog = L.parse_program(g["text"])
    with pytest.raises(P.InterpreterError):
        P.execute(prog, g["binding"], {k: np.array(v) for k, v in g["inputs"].items()})


@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("idx", [1, 3, 9, 13, 17])
@pytest.mark.parametrize("epi", ["relu6", "scale", "scale_bias_relu", "scale_bias_relu6"])
def test_fused_epilogues_on_resnet_layers(P, idx, mode, epi):
    layer = W.LAYERS[idx - 1]
    x, w, b = W.conv_inputs(layer, 2, seed=300 + idx)
    rng = np.random.default_rng(idx)
    s = rng.uniform(0.5, 8.0, layer.K).astype(np.float32)       # pushes values past 6
    kw = dict(stride=layer.stride, pad=layer.pad, mode=mode, channels=layer.C)
    args = {"relu6": dict(bias=b, relu6=True), "scale": dict(scale=s),
            "scale_bias_relu": dict(scale=s, bias=b, relu=True),
            "scale_bias_relu6": dict(scale=s, bias=b, relu6=True)}[epi]
    dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in args.items()}
    X, Wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y = P.conv2d_nchw16c(X, Wt, **dev, **kw)
    conv = oracle.conv2d_f64(x, w, None, stride=layer.stride, pad=layer.pad)
    act = "relu6" if dev.get("relu6") else "relu" if dev.get("relu") else None
    ref = epi_ref(conv, args.get("bias"), args.get("scale"), act)
    scale_ref = np.abs(epi_ref(conv, args.get("bias"), args.get("scale"))).max()
    err = np.abs(y.cpu().numpy().astype(np.float64) - ref).max() / scale_ref
    assert err <= TOL[mode]
    if act == "relu6":
        assert float(y.max()) == 6.0
    # unfused: the same conv, then the stand-alone element-wise kernel -- bitwise, except
    # where the plain conv's default is a 256-column TF32 tile (one accumulation segment;
    # the scale / ReLU6 instances stop at 128 columns)
    y0 = P.conv2d_nchw16c(X, Wt, **kw)
    P.bias_relu_(y0, dev.get("bias"), relu=bool(dev.get("relu")), relu6=bool(dev.get("relu6")),
                 scale=dev.get("scale"))
    if mode == "tf32" and layer.K % 256 == 0 and layer.C_alloc * layer.R * layer.S > 256:
        assert float((y - y0).abs().max()) <= TOL[mode] * scale_ref
    else:
        assert torch.equal(y, y0)


def test_host_path_fused_epilogue_equals_device(P):
    layer = W.LAYERS[7 - 1]
    x, w, b = W.conv_inputs(layer, 3, seed=5)
    s = np.random.default_rng(0).uniform(0.5, 8.0, layer.K).astype(np.float32)
    pw = P.prepack_weights(torch.from_numpy(w).cuda())
    bd, sd = torch.from_numpy(b).cuda(), torch.from_numpy(s).cuda()
    kw = dict(stride=layer.stride, pad=layer.pad, relu6=True, scale=sd, cfg={"split_k": 1})
    dev = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), pw, bd, **kw)
    host = P.conv2d_nchw16c_host(torch.from_numpy(x).pin_memory(), pw, bd, **kw)
    torch.cuda.synchronize()
    assert torch.equal(dev.cpu(), host)


@pytest.mark.parametrize("shape", [(256, 192, 320), (96, 64, 33), (128, 128, 4096), (64, 256, 2048)])
def test_gemm_relu6(P, shape):
    m, n, k = shape
    rng = np.random.default_rng(m)
    a = rng.uniform(-2, 2, (m, k)).astype(np.float32)
    b = rng.uniform(-2, 2, (k, n)).astype(np.float32)
    c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), relu6=True)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    scale = np.abs(ref).max()
    ref = np.where(6.0 < np.where(0.0 > ref, 0.0, ref), 6.0, np.where(0.0 > ref, 0.0, ref))
    assert np.abs(c.cpu().numpy() - ref).max() / scale <= 1e-5
    assert float(c.max()) == 6.0 and float(c.min()) == 0.0


def test_scale_needs_k_values(P):
    x = torch.zeros((1, 1, 4, 4, 16), device="cuda")
    w = torch.zeros((2, 1, 1, 1, 16, 16), device="cuda")
    with pytest.raises(ValueError):
        P.conv2d_nchw16c(x, w, scale=torch.ones(16, device="cuda"))


@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("split_k", [2, 3])
def test_split_k_reduction_applies_extended_epilogue_once(P, mode, split_k):
    """Scale + bias + ReLU6 on the split-K path: partials are written raw, the last
    unit of each tile applies the epilogue once (layer 17 at 2 images: 8 tiles)."""
    layer = W.LAYERS[17 - 1]
    x, w, b = W.conv_inputs(layer, 2, seed=77)
    s = np.random.default_rng(1).uniform(0.5, 8.0, layer.K).astype(np.float32)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode)
    X, bd, sd = (torch.from_numpy(t).cuda() for t in (x, b, s))
    kw = dict(stride=layer.stride, pad=layer.pad, mode=mode, relu6=True, scale=sd)
    y = P.conv2d_nchw16c(X, pw, bd, cfg={"split_k": split_k}, **kw)
    y1 = P.conv2d_nchw16c(X, pw, bd, cfg={"split_k": 1}, **kw)
    conv = oracle.conv2d_f64(x, w, None, stride=layer.stride, pad=layer.pad)
    pre = epi_ref(conv, b, s)
    ref = epi_ref(conv, b, s, "relu6")
    for out in (y, y1):
        assert np.abs(out.cpu().numpy() - ref).max() / np.abs(pre).max() <= TOL[mode]
