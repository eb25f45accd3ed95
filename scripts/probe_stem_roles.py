"""Attribute the ResNet stem's time to pipeline roles with the diagnostic flag
bits (results are wrong when set): each run drops one role's work."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W

L = _lib.lib()
DBG = {"base": 0, "noST": 1 << 9, "noEPI": 1 << 10, "noMMA": 1 << 11, "noGATHER": 1 << 12,
       "noGATHER+noST": (1 << 12) | (1 << 9), "noMMA+noEPI": (1 << 11) | (1 << 10),
       "staging_only": (1 << 11) | (1 << 10), "tma_only": (1 << 12) | (1 << 9) | (1 << 11) | (1 << 10)}
l = W.LAYERS[0]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
b = torch.rand(l.K, device='cuda')
pw = P.prepack_weights(w, channels=l.C)
y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, dbg in DBG.items():
    flags = _lib.PDL_MODE_3XTF32 | _lib.PDL_BIAS | _lib.PDL_RELU | dbg

    def run():
        _lib.check(L.pdl_conv2d_fwd_prepacked(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(pw.data.data_ptr()),
            ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(y.data_ptr()), n, l.C, l.K, l.H, l.W,
            l.R, l.S, l.stride, l.pad, flags, None, st))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    print(f"{l.name()} n={n} {name}: {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)
