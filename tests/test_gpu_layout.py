"""Data path either side of the conv: NCHW <-> nChw16c and
OIHW -> KCRS16c16k pack kernels (bitwise, they only move data), the NCHW
convenience conv, and layer chaining in the blocked layout -- all against
float64 references computed on the CPU."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import paper_2006_02230_b200 as P

pytestmark = pytest.mark.gpu


def _blocked_ref(x):
    n, c, h, w = x.shape
    cb = (c + 15) // 16
    xp = torch.zeros((n, cb * 16, h, w), dtype=x.dtype)
    xp[:, :c] = x
    return xp.reshape(n, cb, 16, h, w).permute(0, 1, 3, 4, 2).contiguous()


@pytest.mark.parametrize("shape", [(2, 3, 7, 9), (1, 16, 13, 13), (3, 40, 5, 300), (2, 64, 56, 56),
                                   (1, 1, 1, 1)])
def test_pack_unpack_roundtrip_bitwise(shape):
    g = torch.Generator().manual_seed(sum(shape))
    x = torch.rand(shape, generator=g) * 2 - 1
    xb = P.to_nchw16c(x.cuda())
    assert torch.equal(xb.cpu(), _blocked_ref(x))
    back = P.from_nchw16c(xb, shape[1])
    assert torch.equal(back.cpu(), x)


def test_pack_weights_bitwise():
    g = torch.Generator().manual_seed(1)
    w = torch.rand((32, 3, 7, 7), generator=g) - 0.5
    wb = P.weights_to_kcrs16c16k(w.cuda()).cpu()
    ref = torch.zeros((32, 16, 7, 7))
    ref[:, :3] = w
    ref = ref.reshape(2, 16, 1, 16, 7, 7).permute(0, 2, 4, 5, 3, 1).contiguous()
    assert torch.equal(wb, ref)


@pytest.mark.parametrize("c,k,h,r,stride,mode,tol", [
    (3, 64, 30, 7, 2, "3xtf32", 1e-5),
    (64, 64, 14, 3, 1, "3xtf32", 1e-5),
    (48, 32, 9, 1, 2, "tf32", 1e-2),
])
def test_conv2d_nchw_matches_fp64(c, k, h, r, stride, mode, tol):
    g = torch.Generator().manual_seed(c + k + h)
    x = torch.rand((2, c, h, h), generator=g) * 2 - 1
    w = torch.rand((k, c, r, r), generator=g) * 2 - 1
    b = torch.rand((k,), generator=g) - 0.5
    y = P.conv2d_nchw(x.cuda(), w.cuda(), b.cuda(), stride=stride, pad=r // 2, relu=True, mode=mode)
    ref = F.relu(F.conv2d(x.double(), w.double(), b.double(), stride=stride, padding=r // 2))
    err = (y.cpu().double() - ref).abs().max() / ref.abs().max()
    assert y.shape == ref.shape and err <= tol, float(err)


def test_layer_chain_stays_blocked():
    """y of one conv is directly the next conv's x (nKhw16k == nChw16c)."""
    g = torch.Generator().manual_seed(7)
    x = torch.rand((2, 32, 16, 16), generator=g) * 2 - 1
    w1 = torch.rand((64, 32, 3, 3), generator=g) - 0.5
    w2 = torch.rand((32, 64, 1, 1), generator=g) - 0.5
    b1, b2 = torch.rand(64, generator=g) - 0.5, torch.rand(32, generator=g) - 0.5
    xb = P.to_nchw16c(x.cuda())
    y1 = P.conv2d_nchw16c(xb, P.weights_to_kcrs16c16k(w1.cuda()), b1.cuda(), pad=1, relu=True)
    y2 = P.conv2d_nchw16c(y1, P.weights_to_kcrs16c16k(w2.cuda()), b2.cuda(), stride=2, relu=True)
    out = P.from_nchw16c(y2, 32).cpu().double()
    r1 = F.relu(F.conv2d(x.double(), w1.double(), b1.double(), padding=1))
    ref = F.relu(F.conv2d(r1, w2.double(), b2.double(), stride=2))
    assert (out - ref).abs().max() / ref.abs().max() <= 1e-5


def test_layout_errors():
    with pytest.raises(P.PdlShapeError):
        P.weights_to_kcrs16c16k(torch.zeros((20, 3, 3, 3), device="cuda"))
