"""Resident-weight 1x1 conv vs the streamed-weight schedule (cluster_m=2)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
for (n, c, k, h) in [(2, 32, 32, 7), (2, 64, 64, 8), (2, 64, 256, 8), (2, 32, 128, 7), (4, 128, 512, 14), (256, 64, 256, 56)]:
    g = torch.Generator(device="cuda").manual_seed(c + k)
    x = torch.rand((n, c // 16, h, h, 16), device="cuda", generator=g) * 2 - 1
    w = torch.rand((k // 16, c // 16, 1, 1, 16, 16), device="cuda", generator=g) - 0.5
    b = torch.rand(k, device="cuda", generator=g) - 0.5
    pw = P.prepack_weights(w)
    ref = P.conv2d_nchw16c(x, pw, b, relu=True, cfg={"cluster_m": 2})
    got = P.conv2d_nchw16c(x, pw, b, relu=True)
    torch.cuda.synchronize()
    d = (got - ref).abs()
    bad = (d > 1e-4).nonzero()
    print(n, c, k, h, "max diff", float(d.max()), "bad", bad.shape[0], bad[:4].tolist() if bad.shape[0] else "", flush=True)
