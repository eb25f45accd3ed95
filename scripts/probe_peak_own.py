"""Tensor-core TF32 throughput of our own tile engine (TF32 mode, 8192^3 GEMM)
and the effect of 64-channel stages (bk=64) on the N=64 conv layers."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W
n = 8192
a = torch.rand(n, n, device='cuda'); b = torch.rand(n, n, device='cuda'); c = torch.empty(n, n, device='cuda')
for mode in ("tf32", "3xtf32"):
    for _ in range(2): P.gemm(a, b, c, mode=mode)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); P.gemm(a, b, c, mode=mode); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"own GEMM 8192^3 {mode}: {2*n**3/best/1e9:.1f} TFLOP/s", flush=True)
for idx in (3, 2, 5):
    l = W.LAYERS[idx - 1]
    x = torch.rand((256, l.C // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C // 16, l.R, l.S, 16, 16), device='cuda')
    bb = torch.rand(l.K, device='cuda')
    y = torch.empty((256, l.K // 16, l.P, l.Q, 16), device='cuda')
    pw = P.prepack_weights(w)
    for bk in (32, 64):
        cfg = {"bk": bk, "cluster_m": 1}
        for _ in range(2): P.conv2d_nchw16c(x, pw, bb, stride=l.stride, pad=l.pad, relu=True, out=y, cfg=cfg)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): P.conv2d_nchw16c(x, pw, bb, stride=l.stride, pad=l.pad, relu=True, out=y, cfg=cfg)
        e1.record(); torch.cuda.synchronize()
        print(f"{l.name()} bk={bk}: {e0.elapsed_time(e1)/5:.4f} ms", flush=True)
