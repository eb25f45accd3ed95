"""Attribute conv time to pipeline roles with diagnostic switches (results are
discarded; the switches break correctness on purpose)."""
import ctypes, json, sys
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W
L = _lib.lib()
DBG = {"base": 0, "noA": 1 << 8, "noST": 1 << 9, "noEPI": 1 << 10, "noA+noST": 3 << 8,
       "noA+noST+noEPI": 7 << 8}
for idx in (1, 3, 7, 4, 17, 9):
    l = W.LAYERS[idx - 1]
    n = 256
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, channels=l.C)
    y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
    out = []
    for name, f in DBG.items():
        flags = _lib.PDL_MODE_3XTF32 | _lib.PDL_BIAS | _lib.PDL_RELU | f
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        def run():
            _lib.check(L.pdl_conv2d_fwd_prepacked(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(pw.data.data_ptr()),
                       ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(y.data_ptr()), n, l.C, l.K, l.H, l.W, l.R, l.S,
                       l.stride, l.pad, flags, None, st))
        for _ in range(2): run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): run()
        e1.record(); torch.cuda.synchronize()
        out.append(f"{name}={e0.elapsed_time(e1)/5:.4f}")
    print(l.name().ljust(24), " ".join(out), flush=True)
