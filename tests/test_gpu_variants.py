"""Every generated tile variant computes the library default's result: within
the mode tolerance always, and bitwise when only bn / cluster differ (the
per-element reduction order depends on bk and on the accumulation segments: 256-column
tiles sum the whole reduction in one)."""
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
    dflt = _lib.default_cfg(_lib.PDL_OP_CONV2D,
                            [2, L.C, L.K, L.H, L.W, L.R, L.S, L.stride, L.pad, _lib.MODES[mode]])
    dflt_bk = 32 if L.C <= 4 else dflt.bk  # the stem ignores bk
    one_seg = L.C_alloc * L.R * L.S <= 256
    bad = []
    for v in vs:
        ok, d = variants.legality_check(L, v, n_images=2, seed=idx, return_detail=True)
        same_order = v.bk == dflt_bk and (one_seg or (v.bn > 128) == (dflt.bn > 128))
        if not ok or (same_order and not d["bitwise"]):
            bad.append((v.vid, d))
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [3, 7, 19])
def test_cta_pair_tiles_bitwise_equal(idx):
    """cluster_n=2: cta_group::2 MMAs over a CTA pair (M=256, B split across the
    pair) give bitwise the single-CTA result (same per-element reduction order)."""
    import torch
    import paper_2006_02230_b200 as P
    from paper_2006_02230_b200.workloads import conv_inputs
    L = LAYERS[idx]
    x, w, b = (torch.from_numpy(t).cuda() for t in conv_inputs(L, 3, seed=idx))
    pw = P.prepack_weights(w, channels=L.C)
    # pairs never split the reduction: compare with the unsplit single-CTA schedule
    ref = P.conv2d_nchw16c(x, pw, b, stride=L.stride, pad=L.pad, relu=True, cfg={"split_k": 1})
    got = P.conv2d_nchw16c(x, pw, b, stride=L.stride, pad=L.pad, relu=True, cfg={"cluster_n": 2})
    assert torch.equal(ref, got)
