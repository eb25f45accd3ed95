"""Small per-GPU batches: schedule options per layer (graph-replayed, isolated)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
idxs = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 6, 10, 11, 16, 18, 20]
for idx in idxs:
    l = W.LAYERS[idx - 1]
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, channels=l.C)
    y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
    menu = [("auto", None), ("s1", {"split_k": 1}), ("s2", {"split_k": 2}), ("s3", {"split_k": 3}),
            ("s4", {"split_k": 4}), ("s6", {"split_k": 6}), ("s8", {"split_k": 8}),
            ("bn64", {"bn": 64}), ("bn64_s1", {"bn": 64, "split_k": 1}),
            ("bn64_s2", {"bn": 64, "split_k": 2})]
    res = []
    for name, cfg in menu:
        def call():
            P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y, cfg=cfg)
        try:
            call()
        except Exception as e:
            res.append(f"{name}=err")
            continue
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    call()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(f"{name}={e0.elapsed_time(e1) / 50 * 1e3:.1f}")
    print(f"n={n} {l.name()}: " + " ".join(res), flush=True)
