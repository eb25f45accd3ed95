"""A/B: cudaLimitMaxL2FetchGranularity (32 / 64 / 128 B) on the stride-2 1x1 layers, whose
parity maps read 64-byte pixels at a 128-byte stride (ncu: 1.6-1.9x the algorithmic DRAM bytes)."""
import ctypes, sys
sys.path.insert(0, '.')
import torch
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W
rt = ctypes.CDLL("libcudart.so.12")
torch.zeros(1, device="cuda")
def time_layer(l, n=256, reps=20):
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, channels=l.C)
    y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
    flush = torch.empty(64 << 20, device='cuda')
    ts = []
    for i in range(reps + 3):
        flush.add_(1.0)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y)
        e.record(); e.synchronize()
        if i >= 3: ts.append(a.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]
for gran in (0, 32, 64, 128):
    if gran:
        rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(gran))
        v = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
        print(f"set granularity {gran}: rc={rc}, now {v.value}")
    else:
        v = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
        print(f"default granularity {v.value}")
    for idx in (6, 11, 16, 9, 7, 4):
        l = W.LAYERS[idx - 1]
        print(f"  {l.name()}: {time_layer(l)*1e3:.1f} us", flush=True)
