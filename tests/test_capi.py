"""CPU-only checks of the C ABI boundary: the library loads, exports every
symbol include/pdl.h declares, and reports a clean error without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2006_02230_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "pdl.h")).read()
    return sorted(set(re.findall(r"\b(pdl_[a-z0-9_]+)\s*\(", txt)))


def test_library_built():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"


def test_exports_match_header():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_abi_version_and_cfg():
    L = _lib.lib()
    assert L.pdl_abi_version() == 1
    cfg = _lib.default_cfg(_lib.PDL_OP_CONV2D, [28, 64, 64, 56, 56, 3, 3, 1, 1, 0])
    assert cfg.bm == 128 and cfg.bn == 64 and cfg.bk == 64   # BN=64 3x3: 64-channel k-blocks
    cfg = _lib.default_cfg(_lib.PDL_OP_CONV2D, [28, 64, 256, 56, 56, 1, 1, 1, 0, 0])
    assert cfg.bn == 128 and cfg.bk == 32
    cfg = _lib.default_cfg(_lib.PDL_OP_GEMM, [4096, 4096, 4096])
    assert cfg.bn in (64, 128, 256)


def test_workspace_and_packed_bytes():
    L = _lib.lib()
    # 3xTF32 carries the hi and lo planes
    assert L.pdl_conv2d_packed_bytes(64, 128, 3, 3, _lib.PDL_MODE_3XTF32) == 2 * 64 * 128 * 9 * 4
    assert L.pdl_conv2d_packed_bytes(64, 128, 3, 3, _lib.PDL_MODE_TF32) == 64 * 128 * 9 * 4
    # ResNet stem (C=3, 7x7): (r, s, c) packed, 2 k-blocks x 20 chunks of 4 values
    assert L.pdl_conv2d_packed_bytes(3, 64, 7, 7, _lib.PDL_MODE_3XTF32) == 2 * 2 * 20 * 64 * 4 * 4
    # other narrow shapes: one k-block (8 taps x 4 channels) per kernel row
    assert L.pdl_conv2d_packed_bytes(4, 64, 7, 7, _lib.PDL_MODE_TF32) == 7 * 8 * 64 * 4 * 4
    assert L.pdl_conv2d_packed_bytes(3, 64, 5, 5, _lib.PDL_MODE_3XTF32) == 2 * 5 * 8 * 64 * 4 * 4
    # a batch that fills the GPU: the workspace is just the packed weights
    dims = (ctypes.c_int * 10)(256, 64, 128, 14, 14, 3, 3, 1, 1, 0)
    assert L.pdl_conv2d_splitk_workspace_bytes(256, 64, 128, 14, 14, 3, 3, 1, 1, 0, None) == 0
    assert L.pdl_workspace_bytes(_lib.PDL_OP_CONV2D, dims, None) == 2 * 64 * 128 * 9 * 4
    # 2 images of 14x14 (3x3, C=256 -> 72 k-blocks of 32 channels) -> 4 tiles of 128 px:
    # split-K x4 (ranges of 18 k-blocks); area = 1 KB of tile counters (fixed) + 4 tiles x
    # 4 ranges x 128 x 128 fp32 partials
    split = 1024 + 4 * 4 * 128 * 128 * 4
    assert L.pdl_conv2d_splitk_workspace_bytes(2, 256, 128, 14, 14, 3, 3, 1, 1, 0, None) == split
    dims = (ctypes.c_int * 10)(2, 256, 128, 14, 14, 3, 3, 1, 1, 0)
    assert L.pdl_workspace_bytes(_lib.PDL_OP_CONV2D, dims, None) == 2 * 256 * 128 * 9 * 4 + split
    # ranges shorter than 16 k-blocks never pay: 64 input channels (18 k-blocks) stay whole
    assert L.pdl_conv2d_splitk_workspace_bytes(2, 64, 128, 14, 14, 3, 3, 1, 1, 0, None) == 0
    # split_k = 1 turns it off; the stem never splits
    off = _lib.TileCfg.make(split_k=1)
    assert L.pdl_conv2d_splitk_workspace_bytes(2, 256, 128, 14, 14, 3, 3, 1, 1, 0, ctypes.byref(off)) == 0
    assert L.pdl_conv2d_splitk_workspace_bytes(1, 3, 64, 224, 224, 7, 7, 2, 3, 0, None) == 0
    # GEMM: 4096^3 fills the GPU; 1024^3 uses 64-column tiles (128 tiles, one wave) and
    # does not split; 512 x 512 x 4096 (32 tiles of 128 x 64, 128 k-blocks) splits x4
    g = (ctypes.c_int * 4)(4096, 4096, 4096, 0)
    assert L.pdl_workspace_bytes(_lib.PDL_OP_GEMM, g, None) == 0
    g = (ctypes.c_int * 4)(1024, 1024, 1024, 0)
    assert L.pdl_workspace_bytes(_lib.PDL_OP_GEMM, g, None) == 0
    g = (ctypes.c_int * 4)(512, 512, 4096, 0)
    assert L.pdl_workspace_bytes(_lib.PDL_OP_GEMM, g, None) == 1024 + 32 * 4 * 128 * 64 * 4


def test_no_gpu_is_a_loud_error():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.lib()
    assert L.pdl_device_check() == _lib.PDL_EDEVICE
    assert b"sm_100" in L.pdl_last_error()
    with pytest.raises(_lib.PdlError):
        _lib.check(L.pdl_gemm_f32(None, None, None, 4, 4, 4, 4, 4, 4, 1.0, 0.0, 0, None, None,
                                  0, None))


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2006_02230_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
