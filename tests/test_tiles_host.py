"""Host-only checks of the conv tile search (pdl_conv2d_schedule runs without a GPU)."""
from paper_2006_02230_b200 import _lib, workloads as W

SINGLE = 8  # PDL_RASTER_SINGLE_IMAGE_TILES
BOX = 2     # PDL_RASTER_BOX_TILES (no segment tiles)


def test_search_fills_more_rows_than_single_image_tiles():
    """Host-only schedule query: the search never has more tiles than the round-1 geometry,
    and has fewer on the 28x28 / 14x14 / 7x7 ResNet layers."""
    fewer = 0
    for n in (256, 32, 28, 1):
        for l in W.LAYERS:
            a = _lib.conv_schedule(n, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0, cfg={"raster": BOX})
            o = _lib.conv_schedule(n, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0, cfg={"raster": BOX | SINGLE})
            assert a["tile_w"] * a["tile_h"] * a["tile_images"] <= 128
            assert a["m_tiles"] <= o["m_tiles"], (n, l.name(), a, o)
            fewer += a["m_tiles"] < o["m_tiles"]
    assert fewer >= 30


def test_explicit_box_is_validated():
    import pytest
    l = W.LAYERS[6]  # 28x28 3x3
    ok = _lib.conv_schedule(9, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0, cfg={"raster": 7 << 8 | 4 << 16 | 4 << 24})
    assert (ok["tile_w"], ok["tile_h"], ok["tile_images"], ok["halo"]) == (7, 4, 4, 1)
    big = _lib.conv_schedule(9, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0, cfg={"raster": 4 << 8 | 4 << 16 | 8 << 24})
    assert big["halo"] == 0  # 6 x 6 x 8 halo pixels do not fit one halo buffer: per-tap boxes
    for bw, bh, bni in ((64, 4, 1), (29, 1, 1), (4, 4, 10), (0, 4, 1)):
        with pytest.raises(_lib.PdlShapeError, match="tile box"):
            _lib.conv_schedule(9, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, 0,
                               cfg={"raster": bw << 8 | bh << 16 | bni << 24})
