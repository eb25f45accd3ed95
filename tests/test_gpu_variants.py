"""Every generated tile variant computes the library default's result: within
the mode tolerance always, and bitwise when only bn / cluster differ (the
per-element reduction order depends on bk alone)."""
import pytest

from paper_2006_02230_b200 import variants, workloads

LAYERS = {L.idx: L for L in workloads.resnet50_v1_layers()}


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [1, 3, 6, 9, 15, 18])
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_all_variants_legal(idx, mode):
    L = LAYERS[idx]
    vs = variants.generate_variants(L, variants.VariantConfig(modes=(mode,)))
    assert vs
    from paper_2006_02230_b200 import _lib
    dflt_bk = _lib.default_cfg(_lib.PDL_OP_CONV2D,
                               [2, L.C, L.K, L.H, L.W, L.R, L.S, L.stride, L.pad, 0]).bk
    if L.C <= 4:
        dflt_bk = 32  # the stem ignores bk
    bad = []
    for v in vs:
        ok, d = variants.legality_check(L, v, n_images=2, seed=idx, return_detail=True)
        if not ok or (v.bk == dflt_bk and not d["bitwise"]):
            bad.append((v.vid, d))
    assert not bad, bad
