"""Time ResNet-50 layers in isolation: flushed single launches (median) and 20 back-to-back launches.
    [PDL_LIB=...] python scripts/time_layer.py [N] [mode] idx [idx ...]"""
import sys
sys.path.insert(0, '.')
import torch
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

N = int(sys.argv[1]); mode = sys.argv[2]
flush = torch.empty(64 << 20, device='cuda')
for idx in [int(a) for a in sys.argv[3:]]:
    l = W.LAYERS[idx - 1]
    x = torch.rand((N, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    if l.C != l.C_alloc:
        x[..., l.C:] = 0
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, mode=mode, channels=l.C)
    y = torch.empty((N, l.K // 16, l.P, l.Q, 16), device='cuda')
    run = lambda: P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, mode=mode, out=y)
    for _ in range(3):
        run()
    ts = []
    for i in range(15):
        flush.add_(1.0)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); e.record(); e.synchronize()
        ts.append(a.elapsed_time(e))
    ts.sort()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        run()
    e.record(); e.synchronize()
    print(f"{l.name()} N={N} {mode}: flushed median {ts[7]*1e3:.1f} us (min {ts[0]*1e3:.1f}, max {ts[-1]*1e3:.1f}); back-to-back {a.elapsed_time(e)/20*1e3:.1f} us", flush=True)
