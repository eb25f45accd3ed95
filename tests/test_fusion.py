"""Alg. 3 fusion pass (paper_2006_02230_b200.fusion) on the CPU.

Fused nests are run by the oracle's IR interpreter (oracle/interp.py, pinned to
the reference's own outputs) and compared bitwise with (a) the reference's
execution of the same fused text and of the unfused program
(tests/golden/fusion_ref.json, tests/golden/gen_fusion.py) and (b) the
reference-made conv -> bias+ReLU goldens."""
import json
import os

import numpy as np
import pytest

from oracle.interp import interpret
from paper_2006_02230_b200 import depend
from paper_2006_02230_b200 import fusion as F
from paper_2006_02230_b200 import loopnest as L

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF = json.load(open(os.path.join(GOLD, "fusion_ref.json")))

GEMM = """param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
gemm: for (i = 0; i < M; i++) {
  for (j = 0; j < N; j++) {
    for (k = 0; k < K; k++) {
      S: C[i][j] += A[i][k] * B[k][j];
    }
  }
}
"""
RELU = """relu: for (i2 = 0; i2 < M; i2++) {
  for (j2 = 0; j2 < N; j2++) {
    R: C[i2][j2] = max(C[i2][j2], 0.0);
  }
}
"""
B = dict(M=3, N=4, K=5)


def pair_of(text, ew_first=False, between=0):
    nests = L.parse_program(text).nests
    if ew_first:
        return F.OperatorPair(nests[1], nests[0], ew_first=True)
    return F.OperatorPair(nests[0], nests[-1], between=tuple(nests[1:len(nests) - 1]))


@pytest.mark.parametrize("case", sorted(REF))
def test_fused_nest_matches_reference_execution(case):
    g = REF[case]
    pair = pair_of(g["text"], g["ew_first"])
    fused = F.fuse(pair, g["binding"])
    assert L.pretty(fused) == g["fused_text"]              # deterministic transformation
    inputs = {k: np.array(v) for k, v in g["inputs"].items()}
    got = interpret(fused, g["binding"], inputs)
    again = interpret(L.parse(g["fused_text"]), g["binding"], inputs)   # text round trip
    for arr, ref in g["fused"].items():
        assert np.array_equal(got[arr], np.array(ref)), arr
        assert np.array_equal(again[arr], np.array(ref)), arr
        assert np.array_equal(np.array(ref), np.array(g["unfused"][arr])), arr  # Alg. 3 invariant


@pytest.mark.parametrize("name", ["conv_1x1_s1_relu", "conv_3x3_s1_relu"])
def test_fused_conv_relu_bitwise_equal_reference_goldens(name):
    d = np.load(os.path.join(GOLD, f"{name}.npz"))
    n, C, K, H, W, R, S, st, pad = (int(d[k]) for k in "N C K H W R S stride pad".split())
    p, q = (H + 2 * pad - R) // st + 1, (W + 2 * pad - S) // st + 1
    hp, wp = st * p - st + R, st * q - st + S
    xp = np.zeros((n, C // 16, hp, wp, 16))
    xp[:, :, pad:pad + H, pad:pad + W, :] = d["x"][:, :, :hp - pad, :wp - pad, :]
    prog = L.parse_program(str(d["text"]))
    b = dict(N=n, KT=K // 16, CT=C // 16, P=p, Q=q, R=R, S=S)
    fused = F.fuse(F.OperatorPair(prog.nests[0], prog.nests[1]), b)
    assert fused.microkernel is None and not fused.has_kernel_call()
    out = interpret(fused, b, {"output": np.zeros((n, K // 16, p, q, 16)), "filter": d["w"],
                               "input": xp, "bias": d["bias"]})
    assert np.array_equal(out["output"], d["y"].ravel())


def test_spec_example_gemm_relu_k4_structure():
    fused = F.fuse(pair_of(GEMM + RELU), dict(M=3, N=4, K=4))
    txt = L.pretty(fused)
    assert "for (k = 0; k < K - 1; k++)" in txt
    assert "S_p1: C[i][j] += A[i][K - 1] * B[K - 1][j];" in txt
    assert "R: C[i][j] = max(C[i][j], 0);" in txt
    # statements: the heavy one, its peeled copy, the element-wise one -- no guards
    assert [s.label for s in fused.statements()] == ["S", "S_p1", "R"]
    info = depend.extract_polyhedral(fused)                 # labels stay unique
    assert [s.label for s in info.statements] == ["S", "S_p1", "R"]


def test_write_set_examples():
    g = L.parse_program(GEMM + RELU).nests
    ws = F.write_set(g[0], B)
    assert set(ws) == {"C"} and len(ws["C"]) == B["M"] * B["N"]
    assert F.write_set(g[1], B) == ws
    col = L.parse("""param M, K;
array C[M][4];
array A[M][K];
w: for (i = 0; i < M; i++) {
  for (k = 0; k < K; k++) {
    S: C[i][0] += A[i][k];
  }
}
""")
    ws = F.write_set(col, dict(M=5, K=3))
    assert ws["C"] == frozenset((i, 0) for i in range(5))


def test_rowsum_is_not_elementwise():
    rowsum = """array r[M];
red: for (i2 = 0; i2 < M; i2++) {
  for (j2 = 0; j2 < N; j2++) {
    R: C[i2][0] += C[i2][j2];
  }
}
"""
    d = F.can_fuse(pair_of(GEMM.replace("array B[K][N];", "array B[K][N];\narray r[M];") + rowsum), B)
    assert not d.fusable and d.failed in (F.WRITE_SETS_DIFFER, F.NOT_ELEMENTWISE)
    # same write set, but a reduction over it
    acc = RELU.replace("R: C[i2][j2] = max(C[i2][j2], 0.0);", "R: C[i2][j2] += C[i2][j2];")
    d = F.can_fuse(pair_of(GEMM + acc), B)
    assert not d.fusable and d.failed == F.NOT_ELEMENTWISE
    # reads a neighbour of the element it writes
    nb = RELU.replace("max(C[i2][j2], 0.0)", "max(C[i2][0], 0.0)")
    d = F.can_fuse(pair_of(GEMM + nb), B)
    assert not d.fusable and d.failed == F.NOT_ELEMENTWISE and d.witness == ("C", (0, 0))


def test_intervening_read_blocks_fusion_with_witness():
    mid = """array z[1];
peek: for (u = 0; u < 1; u++) {
  P: z[u] = C[0][0];
}
"""
    text = GEMM.replace("array B[K][N];", "array B[K][N];\narray z[1];") + mid + RELU
    pair = pair_of(text)
    assert len(pair.between) == 1
    d = F.can_fuse(pair, B)
    assert not d.fusable and d.failed == F.INTERVENING_ACCESS
    assert d.witness[2:] == ("C", (0, 0))
    with pytest.raises(F.FusionError):
        F.fuse(pair, B)


def test_intervening_unrelated_access_is_fine_unless_strict():
    mid = """array bias2[N];
other: for (u = 0; u < N; u++) {
  P: bias2[u] = A[0][0];
}
"""
    ew = RELU.replace("max(C[i2][j2], 0.0)", "max(C[i2][j2] + bias2[j2], 0.0)")
    text = GEMM.replace("array B[K][N];", "array B[K][N];\narray bias2[N];") + mid + ew
    pair = pair_of(text)
    assert F.can_fuse(pair, B).fusable
    d = F.can_fuse(pair, B, strict=True)     # it writes an input of the element-wise op
    assert not d.fusable and d.failed == F.INTERVENING_ACCESS and d.witness[2] == "bias2"


def test_write_sets_differ_witness():
    half = RELU.replace("i2 < M", "i2 < M - 1")
    d = F.can_fuse(pair_of(GEMM + half), B)
    assert not d.fusable and d.failed == F.WRITE_SETS_DIFFER and d.witness == ("C", (2, 0))


def test_triangular_reduction_refused():
    tri = GEMM.replace("for (k = 0; k < K; k++)", "for (k = 0; k < j + 1; k++)")
    d = F.can_fuse(pair_of(tri + RELU), B)
    assert not d.fusable and d.failed == F.NON_RECTANGULAR


@pytest.mark.parametrize("K", [1, 2, 5])
def test_fused_equals_unfused_random(K):
    b = dict(M=4, N=3, K=K)
    text = GEMM + RELU.replace("max(C[i2][j2], 0.0)", "min(max(C[i2][j2], 0.0), 6.0)")
    prog = L.parse_program(text)
    rng = np.random.default_rng(K)
    inputs = {"A": rng.uniform(-3, 3, 4 * K), "B": rng.uniform(-3, 3, K * 3),
              "C": rng.uniform(-3, 3, 12)}
    ref = interpret(prog, b, inputs)
    got = interpret(F.fuse(pair_of(text), b), b, inputs)
    assert np.array_equal(ref["C"], got["C"])


def test_microkernel_band_is_consumed():
    d = np.load(os.path.join(GOLD, "conv_1x1_s1_relu.npz"))
    prog = L.parse_program(str(d["text"]))
    assert prog.nests[0].has_kernel_call()
    b = dict(N=1, KT=1, CT=1, P=2, Q=2, R=1, S=1)
    fused = F.fuse(F.OperatorPair(prog.nests[0], prog.nests[1]), b)
    assert not fused.has_kernel_region() and fused.pair.heavy is prog.nests[0]
    assert L.parse(L.pretty(fused)).statements() == fused.statements()
