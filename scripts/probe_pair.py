"""CTA-pair (cta_group::2) conv tiles vs the single-CTA default: parity + time."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

for arg in sys.argv[1:] or ["7"]:
    l = W.LAYERS[int(arg) - 1]
    n = 256
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device="cuda", generator=g) * 2 - 1
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device="cuda", generator=g) - 0.5
    b = torch.rand(l.K, device="cuda", generator=g) - 0.5
    pw = P.prepack_weights(w, channels=l.C)
    res = {}
    for name, cfg in (("default", None), ("c1", {"cluster_m": 1}), ("pair", {"cluster_n": 2})):
        y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device="cuda")
        run = lambda: P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y, cfg=cfg)
        run()
        torch.cuda.synchronize()
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[name] = (e0.elapsed_time(e1) / 10, y.clone())
    ref = res["default"][1]
    for name, (ms, y) in res.items():
        err = float((y - ref).abs().max() / ref.abs().max())
        print(f"{l.name()} {name:8s} {ms:.4f} ms  max-rel vs default {err:.2e}", flush=True)
