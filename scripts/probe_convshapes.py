"""Implicit-GEMM shapes of ResNet conv layers run as plain GEMMs through the
same tile engine: separates conv-specific costs from shape costs."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W
peak = json.load(open('profiles/peaks_tf32.json'))['tf32_tflops'] * 1e12 / 3
for idx in (3, 7, 12, 17, 9, 19, 13):
    l = W.LAYERS[idx - 1]
    n = 256
    M, N, K = n * l.P * l.Q, l.K, l.C * l.R * l.S
    a = torch.rand(M, K, device='cuda') * 2 - 1
    b = torch.rand(K, N, device='cuda') * 2 - 1
    c = torch.empty(M, N, device='cuda')
    for cl in (1, 2):
        cfg = {"cluster_m": cl}
        for _ in range(3):
            P.gemm(a, b, c, cfg=cfg)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.gemm(a, b, c, cfg=cfg)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        f = 2.0 * M * N * K
        print(f"{l.name():24s} gemm {M}x{N}x{K} cl={cl}: {ms:.4f} ms  {f/ms/1e9:.0f} GF/s  frac {f/(ms/1e3)/peak:.3f}", flush=True)
