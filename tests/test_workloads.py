import numpy as np

from paper_2006_02230_b200 import workloads as W


def test_twenty_distinct_layers_match_survey_appendix_a():
    L = W.LAYERS
    assert len(L) == 20
    assert (L[0].C, L[0].K, L[0].H, L[0].R, L[0].stride, L[0].P) == (3, 64, 224, 7, 2, 112)
    assert sum(l.uses for l in L) == 53
    assert abs(sum(l.flops(28) for l in L) / 1e9 - 77.82) < 0.01
    # spot rows of SURVEY App. A (GFLOP at N=28, MB)
    assert round(L[2].flops(28) / 1e9, 2) == 6.47 and round(L[2].bytes(28) / 1e6, 1) == 45.1
    assert round(L[16].bytes(28) / 1e6, 1) == 15.1
    assert round(L[5].bytes(28) / 1e6, 1) == 33.8  # 1x1 stride-2: x touched = N*C*P*Q


def test_stem_inputs_zero_padded():
    x, w, b = W.conv_inputs(W.LAYERS[0], 1, seed=0)
    assert x.shape == (1, 1, 224, 224, 16)
    assert np.all(x[..., 3:] == 0) and np.all(w[:, :, :, :, 3:, :] == 0)
    assert b.shape == (64,) and np.all(np.abs(b) <= 0.5)


def test_roofline_bound():
    l7 = W.LAYERS[6]
    r = W.Roofline(l7.flops(28), l7.bytes(28), 249e12, 6.5e12)
    assert r.bound == "tensor"
    l2 = W.LAYERS[1]
    assert W.Roofline(l2.flops(28), l2.bytes(28), 249e12, 6.5e12).bound == "hbm"
