"""The interpret()/execute() facade on the GPU: the reference's own .pdl
programs (tests/golden) run end to end and match the reference interpreter's
outputs; tiled / permuted variants give the same result."""
import glob
import os

import numpy as np
import pytest

from paper_2006_02230_b200 import loopnest as L

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(y, ref):
    return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def conv_case(g):
    n, k, c = int(g["N"]), int(g["K"]), int(g["C"])
    stride, pad, r, s = int(g["stride"]), int(g["pad"]), int(g["R"]), int(g["S"])
    p, q = g["y"].shape[2], g["y"].shape[3]
    import oracle
    xp = oracle.pad_nchw16c(g["x"], r, s, stride, pad)
    binding = dict(N=n, KT=k // 16, CT=c // 16, P=int(p), Q=int(q), R=r, S=s)
    inputs = {"input": xp, "filter": g["w"], "output": np.zeros(g["y"].size)}
    if "bias" in g.files:
        inputs["bias"] = g["bias"]
    return binding, inputs


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "conv_*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_interpret_reference_program(path):
    import paper_2006_02230_b200 as P
    g = np.load(path)
    prog = L.parse_program(str(g["text"]))
    binding, inputs = conv_case(g)
    arrays, trace = P.interpret(prog, binding, inputs=inputs)
    from paper_2006_02230_b200.trace import LazyTrace
    assert isinstance(trace, tuple) and len(trace) == len(prog.nests)
    assert all(isinstance(t, LazyTrace) for t in trace)
    assert P.interpret(prog, binding, inputs=inputs, collect_trace=False)[1] is None
    assert rel(arrays["output"].reshape(g["y"].shape), g["y"]) <= 1e-5
    np.testing.assert_array_equal(arrays["filter"], np.asarray(g["w"], np.float64).ravel())


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "gemm_*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_interpret_reference_gemm(path):
    import paper_2006_02230_b200 as P
    g = np.load(path)
    nest = L.parse(str(g["text"]))
    m, n, k = int(g["M"]), int(g["N"]), int(g["K"])
    arrays, trace = P.interpret(nest, dict(M=m, N=n, K=k),
                                inputs={"A": g["A"], "B": g["B"], "C": np.zeros(m * n)})
    assert rel(arrays["C"].reshape(m, n), g["C"]) <= 1e-5
    assert len(trace) == 4 * m * n * k   # A, B, C reads + C write per MAC (simcache.py:193-198)


def test_accumulate_into_nonzero_output_and_tiled_variant():
    import paper_2006_02230_b200 as P
    from test_loopnest import TILED_GEMM, GEMM
    rng = np.random.default_rng(4)
    m, n, k = 16, 12, 32
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    c0 = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    ref = c0.astype(np.float64) + a.astype(np.float64) @ b
    for text in (GEMM, TILED_GEMM):
        out = P.execute(L.parse(text), dict(M=m, N=n, K=k), {"A": a, "B": b, "C": c0})
        assert rel(out["C"].reshape(m, n), ref) <= 1e-5


def test_unfused_bias_relu_nest_alone():
    import paper_2006_02230_b200 as P
    src = """param N, KT, P, Q;
array y[N][KT][P][Q][16];
array bias[KT][16];
e: parallel for (a = 0; a < N; a++) { for (t = 0; t < KT; t++) { for (p = 0; p < P; p++) {
  for (q = 0; q < Q; q++) { for (v = 0; v < 16; v++) {
    T: y[a][t][p][q][v] = max(y[a][t][p][q][v] + bias[t][v], 0.0);
} } } } }
"""
    rng = np.random.default_rng(2)
    y = rng.uniform(-1, 1, (2, 3, 4, 5, 16)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (3, 16)).astype(np.float32)
    out = P.execute(L.parse(src), dict(N=2, KT=3, P=4, Q=5), {"y": y, "bias": bias})
    ref = np.maximum(y.astype(np.float64) + bias[None, :, None, None, :], 0.0)
    assert rel(out["y"].reshape(y.shape), ref) <= 1e-6
