"""The GEMM's fused epilogue (pdl_gemm_f32_epilogue: scale, shift, ReLU / ReLU6 --
the fused GEMM + batch-norm programs of PAPER.md:1228-1241), the conv `+=` path
(pdl_accumulate_epilogue_nchw16c), the executor running GEMM + bnorm + ReLU
programs with no torch element-wise op, flag validation, and library calls on a
side stream (temporaries must live on the stream the kernels run on)."""
import warnings

import numpy as np
import pytest

import oracle
from paper_2006_02230_b200 import loopnest as L
from paper_2006_02230_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = {"3xtf32": 1e-5, "tf32": 1e-2, "fp32": 1e-5}


def rel(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30))


@pytest.fixture(scope="module")
def P():
    import paper_2006_02230_b200 as pkg
    assert pkg.device_ok(), "libpdl.so did not find an sm_100 device"
    return pkg


def gemm_epi_ref(a, b, c0, alpha, beta, scale, bias, act):
    y = alpha * (a.astype(np.float64) @ b.astype(np.float64))
    if c0 is not None:
        y = y + beta * c0.astype(np.float64)
    if scale is not None:
        y = y * scale.astype(np.float64)[None, :]
    if bias is not None:
        y = y + bias.astype(np.float64)[None, :]
    if act in ("relu", "relu6"):
        y = np.where(0.0 > y, 0.0, y)
    if act == "relu6":
        y = np.where(6.0 < y, 6.0, y)
    return y


@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "fp32"])
@pytest.mark.parametrize("shape", [(256, 192, 320), (3136, 64, 576), (49, 2048, 512), (130, 36, 44)])
@pytest.mark.parametrize("epi", ["bias_relu", "bnorm_relu", "bnorm_relu6", "scale", "beta_bias"])
def test_gemm_epilogue(P, mode, shape, epi):
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    a, b = W.gemm_inputs(m, n, k, seed=m)
    bias = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, n).astype(np.float32)
    c0 = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    use_scale = epi.startswith("bnorm") or epi == "scale"
    use_bias = epi != "scale"
    act = "relu6" if epi.endswith("relu6") else ("relu" if "relu" in epi else None)
    beta = 1.0 if epi == "beta_bias" else 0.0
    c = torch.from_numpy(c0).cuda()
    P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), c, beta=beta, mode=mode,
           bias=torch.from_numpy(bias).cuda() if use_bias else None,
           scale=torch.from_numpy(scale).cuda() if use_scale else None,
           relu=act == "relu", relu6=act == "relu6")
    ref = gemm_epi_ref(a, b, c0 if beta else None, 1.0, beta, scale if use_scale else None,
                       bias if use_bias else None, act)
    assert rel(c.cpu().numpy(), ref) <= TOL[mode]


@pytest.mark.parametrize("split", [1, 2, 4])
def test_gemm_epilogue_split_k(P, split):
    m, n, k = 128, 128, 2048
    a, b = W.gemm_inputs(m, n, k, seed=5)
    bias = np.linspace(-0.5, 0.5, n, dtype=np.float32)
    c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), bias=torch.from_numpy(bias).cuda(),
               relu=True, cfg={"split_k": split})
    assert rel(c.cpu().numpy(), gemm_epi_ref(a, b, None, 1, 0, None, bias, "relu")) <= 1e-5


def test_gemm_simt_warning_and_strict(P):
    a, b = W.gemm_inputs(37, 45, 29, seed=1)
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    with pytest.warns(P.ops.SimtPathWarning):
        c = P.gemm(at, bt)
    assert rel(c.cpu().numpy(), oracle.gemm_f64(a, b)) <= 1e-5
    from paper_2006_02230_b200._lib import PdlShapeError
    with pytest.raises(PdlShapeError, match="PDL_NO_SIMT"):
        P.gemm(at, bt, strict=True)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        P.gemm(at, bt, mode="fp32")     # exact-fp32 mode asks for the CUDA cores: no warning


def test_flags_are_validated(P):
    import ctypes
    from paper_2006_02230_b200 import _lib
    L_ = _lib.lib()
    a = torch.zeros((128, 128), device="cuda")
    nul = ctypes.c_void_p(0)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    # PDL_BIAS through the bias-less entry point: EINVAL, nothing silently dropped
    rc = L_.pdl_gemm_f32(p(a), p(a), p(a), 128, 128, 128, 128, 128, 128, 1.0, 0.0, _lib.PDL_BIAS, None,
                         nul, 0, nul)
    assert rc == _lib.PDL_EINVAL
    for bad in (1 << 8, 1 << 12, 1 << 20, 3 << 4):
        rc = L_.pdl_gemm_f32(p(a), p(a), p(a), 128, 128, 128, 128, 128, 128, 1.0, 0.0, bad, None,
                             nul, 0, nul)
        assert rc in (_lib.PDL_EUNSUPPORTED, _lib.PDL_EINVAL), bad
    x = torch.zeros((1, 4, 8, 8, 16), device="cuda")
    w = torch.zeros((4, 4, 1, 1, 16, 16), device="cuda")
    pw = P.prepack_weights(w)
    for bad_raster in (32, 128, 1 << 31):
        with pytest.raises(_lib.PdlShapeError, match="raster"):
            P.conv2d_nchw16c(x, pw, cfg={"raster": bad_raster - (1 << 32) if bad_raster >= 1 << 31 else bad_raster})
    # explicit tile boxes (PDL_RASTER_TILE): more than 128 rows, wider than the map, more images than the batch
    for bw, bh, bni in ((64, 4, 1), (16, 1, 1), (8, 8, 2), (0, 8, 1)):
        with pytest.raises(_lib.PdlShapeError, match="tile box"):
            P.conv2d_nchw16c(x, pw, cfg={"raster": bw << 8 | bh << 16 | bni << 24})
    y = torch.zeros((1, 4, 8, 8, 16), device="cuda")
    rc = L_.pdl_conv2d_fwd_prepacked(p(x), p(pw.data), nul, p(y), 1, 64, 64, 8, 8, 1, 1, 1, 0,
                                     1 << 9, None, nul)
    assert rc == _lib.PDL_EUNSUPPORTED


@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_conv_accumulate_epilogue(P, mode):
    layer = W.ConvLayer(0, 64, 128, 14, 3, 1)
    x, w, b = W.conv_inputs(layer, 2, seed=8)
    y0 = np.random.default_rng(9).uniform(-1, 1, (2, 8, 14, 14, 16)).astype(np.float32)
    y = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), stride=1, pad=1, mode=mode)
    P.accumulate_(y, torch.from_numpy(y0).cuda(), torch.from_numpy(b).cuda(), relu=True)
    ref = oracle.conv2d_f64(x, w, None, stride=1, pad=1) + y0
    ref = np.maximum(ref + b.reshape(1, -1, 1, 1, 16), 0.0)
    assert rel(y.cpu().numpy(), ref) <= TOL[mode]


GEMM_BN = """param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
array s[N];
array t[N];
gemm: for (i = 0; i < M; i++) {
  for (j = 0; j < N; j++) {
    for (k = 0; k < K; k++) {
      S: C[i][j] += A[i][k] * B[k][j];
    }
  }
}
ew: for (i2 = 0; i2 < M; i2++) {
  for (j2 = 0; j2 < N; j2++) {
    E: C[i2][j2] = max(C[i2][j2] * s[j2] + t[j2], 0.0);
  }
}
"""


@pytest.mark.parametrize("c_nonzero", [False, True])
def test_executor_gemm_bnorm_relu_on_tensor_cores(P, c_nonzero, monkeypatch):
    """GEMM + batch-norm + ReLU program at a tensor-core shape: one repo kernel with
    the fused epilogue (beta = 1 when C comes in non-zero), no torch element-wise op."""
    m, n, k = 256, 192, 320
    a, b = W.gemm_inputs(m, n, k, seed=11)
    rng = np.random.default_rng(12)
    s = rng.uniform(0.5, 1.5, n).astype(np.float32)
    t = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    c0 = rng.uniform(-1, 1, (m, n)).astype(np.float32) if c_nonzero else np.zeros((m, n), np.float32)
    calls = []
    import paper_2006_02230_b200.ops as ops
    real = ops.gemm
    monkeypatch.setattr(ops, "gemm", lambda *aa, **kw: calls.append(kw) or real(*aa, **kw))
    for name in ("where", "add", "mul"):   # any torch element-wise op on the path fails the test
        monkeypatch.setattr(torch, name, lambda *aa, **kw: (_ for _ in ()).throw(AssertionError(name)))
    out = P.execute(L.parse_program(GEMM_BN), dict(M=m, N=n, K=k),
                    {"A": a, "B": b, "C": c0, "s": s, "t": t})
    assert len(calls) == 1 and calls[0]["beta"] == (1.0 if c_nonzero else 0.0)
    ref = np.maximum((c0.astype(np.float64) + a.astype(np.float64) @ b) * s + t, 0.0)
    assert rel(out["C"].reshape(m, n), ref) <= 1e-5


def test_side_stream_temporaries(P):
    """conv with a fused scale (a temporary [shift | scale] buffer), split-K (a zeroed
    workspace) and the NCHW convenience path (three intermediates), all on a side
    stream while the current stream is busy: results equal the current-stream ones."""
    layer = W.ConvLayer(0, 512, 512, 7, 3, 1)
    x, w, b = W.conv_inputs(layer, 4, seed=13)
    xt, wt, bt = (torch.from_numpy(v).cuda() for v in (x, w, b))
    sc = torch.linspace(0.5, 1.5, 512, device="cuda")
    pw = P.prepack_weights(wt)
    ref = P.conv2d_nchw16c(xt, pw, bt, stride=1, pad=1, relu=True, scale=sc, cfg={"split_k": 2})
    xn = torch.rand((2, 3, 20, 20), device="cuda")
    wn = torch.rand((32, 3, 3, 3), device="cuda")
    ref2 = P.conv2d_nchw(xn, wn, pad=1)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    torch.cuda._sleep(50_000_000)          # keep the current stream busy meanwhile
    outs = []
    for _ in range(3):
        outs.append(P.conv2d_nchw16c(xt, pw, bt, stride=1, pad=1, relu=True, scale=sc,
                                     cfg={"split_k": 2}, stream=side))
        outs.append(P.conv2d_nchw(xn, wn, pad=1, stream=side))
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert torch.equal(o, ref if i % 2 == 0 else ref2)
