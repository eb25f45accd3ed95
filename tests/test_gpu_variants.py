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
    dflt_bk = 32 if ((L.C + 15) // 16) % 2 == 0 else 16
    bad = []
    for v in vs:
        ok, d = variants.legality_check(L, v, n_images=2, seed=idx, return_detail=True)
        if not ok or (v.bk == dflt_bk and not d["bitwise"]):
            bad.append((v.vid, d))
    assert not bad, bad
