"""Ranking path on the CPU: Alg. 1 working sets (pinned to the reference),
Alg. 2 placement, Eq. 1 cost, the DNN judge and the tile-variant generator."""
import json
import os
import sys
import warnings
from fractions import Fraction

import numpy as np
import pytest

from paper_2006_02230_b200 import machine as M
from paper_2006_02230_b200 import rank as R
from paper_2006_02230_b200 import variants as V
from paper_2006_02230_b200 import workloads
from paper_2006_02230_b200.loopnest import UnboundParameterError, parse
from paper_2006_02230_b200.wset import WorkingSetError, working_sets

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF_SRC)

MATMUL = """param M, N, K;
array C[M][N]; array A[M][K]; array B[K][N];
mm: for (i = 0; i < M; i++) {
  for (j = 0; j < N; j++) {
    for (k = 0; k < K; k++) {
      S: C[i][j] += A[i][k] * B[k][j];
} } }
"""


def _entries(rep):
    return sorted([e.dep_id, e.kind, e.array, e.variant, e.elements] for e in rep.entries)


# ----------------------------------------------------------------------------- Alg. 1
@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "wset_ref.json")))["cases"],
                         ids=lambda c: c["name"])
def test_working_sets_match_reference_goldens(case):
    rep = working_sets(parse(case["text"]), case["binding"])
    assert _entries(rep) == sorted(case["entries"])


@pytest.mark.parametrize("m,n,k", [(4, 4, 4), (8, 6, 5), (16, 16, 16), (5, 7, 11)])
def test_worked_example_closed_forms(m, n, k):
    """d2 on A[i][k] has WS_min = 2K+3, WS_max = NK+N+1."""
    rep = working_sets(parse(MATMUL), {"M": m, "N": n, "K": k})
    d = {e.key(): e.elements for e in rep.entries if e.array == "A"}
    assert d["S:r0->S:r0:min"] == 2 * k + 3
    assert d["S:r0->S:r0:max"] == n * k + n + 1


def test_working_sets_min_le_max_and_parallel_entry():
    rep = working_sets(parse(MATMUL.replace("mm: for", "mm: parallel for")), {"M": 4, "N": 3, "K": 5})
    by = {}
    for e in rep.entries:
        by.setdefault(e.dep_id, {})[e.variant] = e.elements
    assert any("par" in v for v in by.values())
    for v in by.values():
        assert ("par" in v) != ("min" in v)
        if "min" in v:
            assert v["min"] <= v["max"]
    par = [e for e in rep.entries if e.variant == "par"][0]
    assert par.array == "B" and par.elements == 4 * 3 + 4 * 5 + 5 * 3  # all i: every element


def test_working_sets_errors_and_empty():
    with pytest.raises(UnboundParameterError):
        working_sets(parse(MATMUL), {"M": 2, "N": 2})
    with pytest.raises(WorkingSetError):
        working_sets(parse(MATMUL), {"M": 64, "N": 64, "K": 64}, limit=1000)
    assert working_sets(parse(MATMUL), {"M": 0, "N": 2, "K": 2}).entries == ()
    rep = working_sets(parse(MATMUL), {"M": 2, "N": 2, "K": 2})
    assert rep.to_dict()["summary"]["entries"] == len(rep.entries)


@pytest.mark.skipif(not HAVE_REF, reason="reference sources only in the build container")
def test_working_sets_live_against_reference():
    sys.path.insert(0, REF_SRC)
    try:
        from looprank import loopdsl, wset
    finally:
        sys.path.remove(REF_SRC)
    text = MATMUL.replace("mm: for", "mm: parallel for")
    for b in ({"M": 2, "N": 3, "K": 2}, {"M": 3, "N": 2, "K": 4}):
        ref = wset.working_sets(loopdsl.parse(text), b)
        assert _entries(working_sets(parse(text), b)) == _entries(ref)


# ----------------------------------------------------------------------------- machine / Alg. 2
def test_default_machine_and_invariants():
    m = M.default_machine()
    assert m.level_names() == ["SMEM", "TMEM", "L2"] and m.cores == 148
    e = M.effective_sizes(m, 148)
    assert e.levels[2].size == m.levels[2].size // 148 and e.levels[0].size == m.levels[0].size
    d = M.machine_to_dict(m)
    assert M.machine_from_dict(d) == m
    bad = dict(d, levels=[d["levels"][1], d["levels"][0], d["levels"][2]])
    with pytest.raises(M.MachineError):
        M.machine_from_dict(bad)
    bad = dict(d, memory={"latency": 1, "bandwidth": 1})
    with pytest.raises(M.MachineError):
        M.machine_from_dict(bad)
    with pytest.raises(M.MachineError):
        M.machine_from_dict({"levels": []})


def test_assign_to_caches_greedy_smallest_first():
    m = M.MachineModel("toy", (M.CacheLevel("L1", 100, 4, 64.0), M.CacheLevel("L2", 1000, 12, 32.0)),
                       100, 8.0, dtype_size=4)

    class E:
        def __init__(self, k, n):
            self.k, self.elements = k, n

        def key(self):
            return self.k

    class Rep:
        entries = [E("a", 20), E("b", 10), E("c", 250), E("d", 30), E("e", 10)]

    a = M.assign_to_caches(Rep, m)
    where = dict(a.placements)
    # bytes: b=40, e=40 -> L1 (80); a=80 -> L2; d=120 -> L2; c=1000 -> L2 has 800 left -> mem
    assert where == {"b": "L1", "e": "L1", "a": "L2", "d": "L2", "c": "mem"}
    assert a.level_total("L1") == 80 and a.level_total("L2") == 200 and a.mem_bytes == 1000
    c = R.cost(a, m)
    assert c == Fraction(80 * 4, 64) + Fraction(200 * 12, 32) + Fraction(1000 * 100, 8)


# ----------------------------------------------------------------------------- Eq. 1 / DNN
def _toy_stats(rng, n):
    return [R.VariantStats(f"v{i:02d}", *rng.integers(0, 10_000, size=4).astype(float)) for i in range(n)]


def test_rank_by_cost_exact_and_tiebreak():
    m = M.default_machine()
    s = [R.VariantStats("b", 1, 2, 3, 4), R.VariantStats("a", 1, 2, 3, 4), R.VariantStats("c", 0, 0, 0, 1)]
    r = R.rank_by_cost(s, m)
    assert r.order == ("c", "a", "b")
    assert R.cost_of_stats(s[2], m) == Fraction(600) / Fraction(22)
    with pytest.raises(R.RankError):
        R.rank_by_cost([], m)


def test_pair_features_joint_normalisation():
    a, b = R.VariantStats("a", 1, 1, 0, 2), R.VariantStats("b", 0, 0, 0, 4)
    f = R.pair_features(a, b)
    assert f.shape == (8,) and abs(f.sum() - 1) < 1e-12 and f[7] == 0.5
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        z = R.pair_features(R.VariantStats("x", 0, 0, 0, 0), R.VariantStats("y", 0, 0, 0, 0))
    assert np.allclose(z, 0.125) and w


def test_model_save_load_judge_tournament(tmp_path):
    m = R.RankerModel.initialize(seed=3)
    assert [w.shape for w in m.weights] == [(64, 8), (32, 64), (16, 32), (8, 16), (2, 8)]
    p = tmp_path / "m.npz"
    m.save(str(p))
    m2 = R.RankerModel.load(str(p))
    x = np.random.default_rng(0).random((5, 8))
    assert np.array_equal(m.forward_batch(x), m2.forward_batch(x))
    stats = _toy_stats(np.random.default_rng(1), 6)
    t1, t2 = R.tournament_rank(m, stats), R.tournament_rank(m2, list(reversed(stats)))
    assert t1 == t2 and sorted(t1.order) == sorted(s.variant_id for s in stats)
    assert R.dnn_judge(m, stats[0], stats[1]) in ("win1", "win2", "draw")
    with pytest.raises(R.RankError):
        R.tournament_rank(m, stats[:1])


def test_gradients_match_finite_differences():
    rng = np.random.default_rng(0)
    m = R.RankerModel.initialize(seed=1)
    X = rng.random((7, 8))
    y = rng.integers(0, 2, size=7)
    loss, gw, gb, _ = R.loss_and_gradients(m, X, y)
    for layer in (0, 2, 4):
        for (r, c) in ((0, 0), (1, 3)):
            old = m.weights[layer][r, c]
            m.weights[layer][r, c] = old + 1e-6
            lp = R.loss_and_gradients(m, X, y)[0]
            m.weights[layer][r, c] = old - 1e-6
            lm = R.loss_and_gradients(m, X, y)[0]
            m.weights[layer][r, c] = old
            assert abs((lp - lm) / 2e-6 - gw[layer][r, c]) < 1e-5


def _separable(n, seed=0):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        a, b = _toy_stats(rng, 2)
        rows.append((a, b, 0 if a.ws_mem < b.ws_mem else 1))
    return rows


def test_train_ranker_deterministic_and_learns(tmp_path):
    data = _separable(300)
    cfg = R.TrainConfig(epochs=300, seed=5)
    r1, r2 = R.train_ranker(data, cfg), R.train_ranker(data, cfg)
    assert all(np.array_equal(a, b) for a, b in zip(r1.model.weights, r2.model.weights))
    assert r1.train_accuracy > 0.85 and r1.val_accuracy > 0.8
    path = tmp_path / "d.csv"
    R.save_dataset(str(path), data[:10])
    back = R.load_dataset(str(path))
    assert [lab for *_, lab in back] == [lab for *_, lab in data[:10]]
    assert np.array_equal(back[3][0].vector(), data[3][0].vector())
    with pytest.raises(R.RankError):
        R.train_ranker([])
    with pytest.raises(R.RankError):
        R.train_ranker([(data[0][0], data[0][1], 2)])


@pytest.mark.skipif(not HAVE_REF, reason="reference sources only in the build container")
def test_training_bitwise_equal_to_reference():
    sys.path.insert(0, REF_SRC)
    try:
        from looprank import rank as ref
    finally:
        sys.path.remove(REF_SRC)
    data = _separable(120, seed=2)
    mine = R.train_ranker(data, R.TrainConfig(epochs=15, seed=4))
    rd = [(ref.VariantStats(a.variant_id, a.ws_l1, a.ws_l2, a.ws_l3, a.ws_mem),
           ref.VariantStats(b.variant_id, b.ws_l1, b.ws_l2, b.ws_l3, b.ws_mem), lab)
          for a, b, lab in data]
    theirs = ref.train_ranker(rd, ref.TrainConfig(epochs=15, seed=4))
    for a, b in zip(mine.model.weights, theirs.model.weights):
        assert np.allclose(a, b, rtol=0, atol=1e-12)
    assert mine.val_accuracy == theirs.val_accuracy


def test_kendall_tau():
    assert R.kendall_tau("abcd", "abcd") == 1.0
    assert R.kendall_tau("abcd", "dcba") == -1.0
    assert R.kendall_tau(["a", "b", "c"], ["b", "a", "c"]) == pytest.approx(1 / 3)


# ----------------------------------------------------------------------------- variants
def test_variants_deterministic_and_legal():
    layers = workloads.resnet50_v1_layers()
    for L in layers:
        vs = V.generate_variants(L)
        assert vs == V.generate_variants(L) and vs, L.name()
        assert [v.vid for v in vs] == sorted(v.vid for v in vs)
        for v in vs:
            assert V.legal(L, v)
            cfg = V.emit_launch(v)
            assert cfg["bn"] in (64, 128, 256) and cfg["bk"] in (16, 32, 64)
            if (L.C // 16) % 2 == 0:
                assert v.cg >= 2
    stem = layers[0]
    assert [v.vid for v in V.generate_variants(stem)] == ["bn64_bk32_c1_3xtf32"]
    both = V.generate_variants(layers[5], V.VariantConfig(modes=("3xtf32", "tf32")))
    assert {v.mode for v in both} == {"3xtf32", "tf32"}


def test_engine_geometry_matches_host_rules():
    L = workloads.ConvLayer(2, 64, 64, 56, 1, 1, 1)  # 1x1 s1 56x56: flattened to 3136 px rows
    g = V.engine_geometry(L, V.TileVariant("x", 64, 32, 1), 256)
    assert g["flat"] and g["bw"] == 128 and g["bh"] == 1 and g["m_tiles"] == 25 * 256
    L3 = workloads.ConvLayer(18, 512, 512, 7, 3, 1, 1)  # 7x7 3x3: one row of 18 images per tile (126 rows)
    g = V.engine_geometry(L3, V.TileVariant("x", 128, 32, 1), 256)
    assert (g["bw"], g["bh"], g["bni"], g["rows_valid"], g["halo"]) == (7, 1, 18, 126, 0)
    assert g["num_kb"] == (512 // 32) * 9
    # the round-1 geometry: whole images, 2 per tile (98 rows), halo mode
    g = V.engine_geometry(L3, V.make_variant(128, 32, 1, tile="single"), 256)
    assert (g["bw"], g["bh"], g["bni"], g["rows_valid"], g["halo"]) == (7, 7, 2, 98, 1)
    g = V.engine_geometry(L3, V.make_variant(128, 32, 1, tile="7x2x9"), 256)
    assert (g["bw"], g["bh"], g["bni"], g["rows_valid"]) == (7, 2, 9, 126)


def test_b200_stats_and_model_rank():
    L = workloads.resnet50_v1_layers()[3]
    vs = V.generate_variants(L)
    stats = [R.stats_for_variant(L, v, 256) for v in vs]
    assert all(s.ws_l1 > 0 and s.ws_l3 > 0 for s in stats)
    r = R.rank_by_model(L, vs, 256)
    assert sorted(r.order) == sorted(v.vid for v in vs)
    assert all(s > 0 for _, s in r.scores)


def test_fitted_artifacts_and_choose_variant():
    """The shipped pipeline model / judge load, and every ranking method picks
    a legal variant deterministically."""
    pm = R.PipelineModel.load()
    assert pm.fitted_on != "defaults"
    L = workloads.resnet50_v1_layers()[16]
    for meth in ("dnn", "model", "cost"):
        v = R.choose_variant(L, 256, "3xtf32", method=meth)
        assert V.legal(L, v) and v == R.choose_variant(L, 256, "3xtf32", method=meth)
    st = pm.term_stats(L, v, 256)
    assert min(st.vector()) >= 0 and st.ws_l1 > 0
    with pytest.raises(R.RankError):
        R.choose_variant(L, 256, method="nope")
    assert R.choose_variant(workloads.resnet50_v1_layers()[0], 256).vid == "bn64_bk32_c1_3xtf32"


def test_ranker_report_committed():
    rep = json.load(open(os.path.join(os.path.dirname(__file__), "..", "profiles", "ranker_r1.json")))
    assert rep["model_loo"]["top1_regret_mean"] < rep["eq1_cost"]["top1_regret_mean"]
    assert rep["dnn_pipeline_terms"]["heldout_accuracy"] > 0.8


# ----------------------------------------------------------------------------- R1-R3, R5
@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "wset_ref.json")))["cases"],
                         ids=lambda c: c["name"])
def test_dependences_and_domains_match_reference(case):
    from paper_2006_02230_b200 import depend as D
    info = D.extract_polyhedral(parse(case["text"]))
    b = case["binding"]
    deps = [D.classify_parallel_span(d, info, b) for d in D.compute_dependences(info, b)]
    assert sorted([d.dep_id, d.kind, d.array, d.spans_parallel, d.parallel_iterator] for d in deps) == \
        sorted(case["deps"])
    for label, dom in case["domains"].items():
        assert D.domain_size(info, label, b) == dom["cardinality"]
        lo, hi = D.domain_lexmin(info, label, b), D.domain_lexmax(info, label, b)
        if dom["lexmin"] is None:
            assert lo is None
        else:
            assert [lo[v] for v in dom["vars"]] == dom["lexmin"]
            assert [hi[v] for v in dom["vars"]] == dom["lexmax"]


# ----------------------------------------------------------------------------- tile form vs Alg. 1
@pytest.mark.parametrize("tiles", [(2, 2, 2, 4, 4, 4), (2, 3, 2, 4, 6, 6), (3, 2, 2, 6, 4, 6),
                                   (2, 2, 3, 4, 4, 9), (4, 2, 2, 8, 4, 4), (1, 4, 2, 2, 8, 6)])
def test_engine_nest_working_sets_closed_form_vs_alg1(tiles):
    """The tile engine's schedule written as a loop nest, enumerated by Alg. 1
    (wset.working_sets, pinned to the reference) at desk-size bindings, equals the
    closed forms the B200 tile working sets are built from."""
    from paper_2006_02230_b200 import wset as WS
    bm, bn, bk, M, N, K = tiles
    enum = WS.working_sets(parse(WS.engine_gemm_nest(bm, bn, bk)), dict(M=M, N=N, K=K))
    closed = WS.engine_gemm_working_sets(bm, bn, bk, M, N, K)
    key = lambda e: (e.dep_id, e.variant)  # noqa: E731
    assert sorted((key(e), e.elements) for e in enum.entries) == \
        sorted((key(e), e.elements) for e in closed.entries)


def test_tile_working_sets_leading_terms_match_closed_form():
    """At BASELINE sizes the tile form's accumulator + panel entries are the leading
    terms of Alg. 1's accumulator working set of the engine nest."""
    from paper_2006_02230_b200 import wset as WS
    for (m, n, k) in [(1024, 1024, 1024), (4096, 4096, 4096), (3136, 64, 576)]:
        g = workloads.GemmShape(m, n, k)
        for v in V.generate_variants(g):
            rep = {e.dep_id: e.elements for e in WS.tile_working_sets(g, v, 1).entries}
            closed = WS.engine_gemm_working_sets(128, v.bn, 32, m, n, k)
            c_max = next(e.elements for e in closed.entries if e.array == "C" and e.variant == "max")
            lead = rep["tmem.acc"] // 2 + rep["l2.Apanel"] + rep["l2.Bpanel"]
            assert c_max == lead - (128 + v.bn) * 32 + 2 * 32, (m, n, k, v.vid)
