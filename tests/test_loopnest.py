"""The .pdl front end (host mirror of looprank.loopdsl) and the executor's
nest recognition -- CPU only (recognition does not launch kernels)."""
import glob
import os

import numpy as np
import pytest

from paper_2006_02230_b200 import loopnest as L
from paper_2006_02230_b200.executor import (ConvPlan, EltwisePlan, GemmPlan, InterpreterError,
                                            make_inputs, plan_program)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GEMM = """param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
gemm: parallel for (i = 0; i < M; i++) {
  for (j = 0; j < N; j++) {
    for (k = 0; k < K; k++) {
      S: C[i][j] += A[i][k] * B[k][j];
    }
  }
}
"""


def test_parse_gemm_structure():
    n = L.parse(GEMM)
    assert n.name == "gemm" and n.params == ("M", "N", "K")
    loops = n.loops()
    assert [lp.iterator for lp in loops] == ["i", "j", "k"]
    assert loops[0].parallel and not loops[1].parallel
    st = n.statements()[0]
    assert st.label == "S" and st.op == "+="
    # `+=` reads the target after the expression operands (loopdsl.py:102-108)
    assert [a.array for a in st.read_accesses()] == ["A", "B", "C"]
    assert n.shapes({"M": 3, "N": 4, "K": 5}) == {"C": (3, 4), "A": (3, 5), "B": (5, 4)}


def test_pretty_roundtrip():
    n = L.parse(GEMM)
    n2 = L.parse(L.pretty(n))
    assert n2 == n
    assert L.to_json(n)["version"] == 1


@pytest.mark.parametrize("src,where", [
    ("param N; array A[N]; x: for (i = 0; i < N; i++) { A[i*i] = 1.0; }", "non-affine"),
    ("param N; array A[N]; x: for (i = 0; i < N; j++) { A[i] = 1.0; }", "increment"),
    ("param N; array A[N]; x: for (i = 0; i < N; i++) { A[i] = alpha; }", "scalar operand"),
    ("param N; array A[N]; x: for (i = 0; i < N; i++) { }", "empty loop body"),
    ("param N; array A[N]; x: for (i = 0; i < N; i++) { A[i] = 1.0 $ }", "unexpected character"),
    ("param N; array A[N]; #pragma foo\nx: for (i = 0; i < N; i++) { A[i] = 1.0; }", "malformed pragma"),
])
def test_parse_errors_carry_position(src, where):
    with pytest.raises(L.ParseError) as ei:
        L.parse(src)
    assert where in str(ei.value)
    assert ei.value.line >= 1 or "expected" in str(ei.value)


def test_non_affine_is_typed():
    with pytest.raises(L.NonAffineError):
        L.parse("param N; array A[N]; x: for (i = 0; i < N; i++) { A[i*i] = 1.0; }")


def test_derived_iterator_folded():
    n = L.parse("param P; array y[P]; array x[2*P]; c: for (oj = 0; oj < P; oj++) "
                "{ ij = oj * 2; y[oj] += x[ij + 1]; }")
    st = n.statements()[0]
    assert st.read_accesses()[0].indices[0] == L.Affine({"oj": 2}, 1)


def conv_text(path):
    return str(np.load(path)["text"])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "conv_*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_golden_programs_parse_and_plan(path):
    g = np.load(path)
    prog = L.parse_program(str(g["text"]))
    nest = prog.nests[0]
    assert nest.microkernel is not None and nest.has_kernel_call()
    sub = L.substitute_microkernel(nest)
    assert sub.has_kernel_region() and not sub.has_kernel_call()
    assert L.reinstate_microkernel(sub) == nest
    binding = dict(N=int(g["N"]), KT=int(g["K"]) // 16, CT=int(g["C"]) // 16,
                   P=int(g["y"].shape[2]), Q=int(g["y"].shape[3]), R=int(g["R"]), S=int(g["S"]))
    plans = plan_program(prog.nests, binding)
    assert len(plans) == 1 and isinstance(plans[0], ConvPlan)
    pl = plans[0]
    assert pl.stride == int(g["stride"]) and pl.parallel_role == "img"
    assert (pl.epilogue is not None) == bool(g["relu"])
    if pl.epilogue is not None:
        assert pl.epilogue.relu and pl.epilogue.bias == "bias"


def test_reinstate_refuses_modified_band():
    g = np.load(os.path.join(GOLD, "conv_3x3_s1.npz"))
    nest = L.parse(str(g["text"]))
    sub = L.substitute_microkernel(nest)
    from dataclasses import replace
    bad = replace(sub, body=L.rebuild(sub.body, lambda n: L.KernelRegion(n.name, n.args, n.body[:0] or n.body[0].body)
                                       if isinstance(n, L.KernelRegion) else n))
    with pytest.raises(L.LoopDslError):
        L.reinstate_microkernel(bad)


TILED_GEMM = """param M, N, K;
array C[M][N]; array A[M][K]; array B[K][N];
g: parallel for (it = 0; it < M; it += 4) {
  for (kt = 0; kt < K; kt += 8) {
    for (j = 0; j < N; j++) {
      for (ii = 0; ii < 4; ii++) {
        for (kk = 0; kk < 8; kk++) {
          S: C[it + ii][j] += B[kt + kk][j] * A[it + ii][kt + kk];
} } } } }
"""


def test_tiled_permuted_gemm_recognised():
    n = L.parse(TILED_GEMM)
    plans = plan_program([n], {"M": 16, "N": 12, "K": 32})
    assert isinstance(plans[0], GemmPlan)
    assert (plans[0].M, plans[0].N, plans[0].K) == (16, 12, 32)
    assert plans[0].parallel_role == "i"


def test_overlapping_tiles_rejected():
    src = TILED_GEMM.replace("ii < 4", "ii < 5")  # tiles overlap: not a GEMM any more
    with pytest.raises(InterpreterError):
        plan_program([L.parse(src)], {"M": 16, "N": 12, "K": 32})


def test_unsupported_nest_raises():
    src = "param N; array A[N]; array B[N]; t: for (i = 0; i < N; i++) { B[i] = A[i] * A[i]; }"
    with pytest.raises(InterpreterError):
        plan_program([L.parse(src)], {"N": 8})


def test_gemm_relu_fused_plan():
    src = GEMM + """relu: for (i2 = 0; i2 < M; i2++) { for (j2 = 0; j2 < N; j2++) {
      T: C[i2][j2] = max(C[i2][j2], 0.0); } }
"""
    prog = L.parse_program(src)
    plans = plan_program(prog.nests, {"M": 4, "N": 4, "K": 4})
    assert len(plans) == 1 and plans[0].epilogue is not None and plans[0].epilogue.relu


def test_make_inputs_matches_reference_streams():
    n = L.parse(GEMM)
    a = make_inputs(n, {"M": 2, "N": 3, "K": 4}, seed=5)
    rng = np.random.default_rng(5)
    for name in sorted(a):
        assert np.array_equal(a[name], rng.standard_normal(a[name].size))


REF = "/root/reference/pkg/src"


def _ref_loopdsl():
    if not os.path.isdir(REF):
        pytest.skip("reference tree not present (GPU box)")
    import importlib
    import sys
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    return importlib.import_module("looprank.loopdsl")


def _canon_aff(a):
    # reference AffineExpr: .coeffs / .const ; ours: .terms / .c0
    coeffs = getattr(a, "coeffs", None)
    if coeffs is None:
        return (tuple(sorted(a.terms.items())), a.c0)
    return (tuple(sorted(coeffs.items())), a.const)


def _canon(nest):
    out = []
    for lp in nest.loops():
        out.append(("loop", lp.iterator, _canon_aff(lp.lower), tuple(_canon_aff(u) for u in lp.upper),
                    lp.step, lp.parallel))
    for st in nest.statements():
        accs = (st.target,) + tuple(st.read_accesses())
        out.append(("stmt", st.label, st.op,
                    tuple((a.array, a.kind, tuple(_canon_aff(i) for i in a.indices)) for a in accs)))
    out.append(("arrays", tuple((n, tuple(_canon_aff(d) for d in dims)) for n, dims in nest.arrays)))
    return out


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_parser_agrees_with_reference_parser(path):
    ref = _ref_loopdsl()
    text = str(np.load(path)["text"])
    mine = L.parse_program(text)
    theirs = ref.parse_program(text)
    assert len(mine.nests) == len(theirs.nests)
    for a, b in zip(mine.nests, theirs.nests):
        assert a.name == b.name
        assert _canon(a) == _canon(b)
        assert _canon(L.substitute_microkernel(a)) == _canon(ref.substitute_microkernel(b))
