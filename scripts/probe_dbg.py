"""Time one conv layer with diagnostic flags that switch pipeline pieces off
(DBG_* in csrc/pdl_kernels.cuh) to find the binding resource."""
import ctypes, sys
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W
lib = _lib.lib()
FL = {"none": 0, "noA": 1 << 8, "noST": 1 << 9, "noEPI": 1 << 10, "noMMA": 1 << 11, "noLOAD": 1 << 12}
combos = ["none", "noLOAD", "noST", "noEPI", "noMMA", "noMMA+noST", "noLOAD+noST+noEPI", "noMMA+noEPI",
          "noA", "noA+noST"]
for arg in sys.argv[1:] or ["1"]:
    l = W.LAYERS[int(arg) - 1]
    n = 256
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, channels=l.C)
    y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
    for cmb in combos:
        fl = 3 | sum(FL[c] for c in cmb.split("+"))  # bias + relu, 3xTF32
        def run():
            rc = lib.pdl_conv2d_fwd_prepacked(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(pw.data.data_ptr()),
                                              ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                              n, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, fl, None,
                                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            assert rc == 0, _lib.lib().pdl_last_error()
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"{l.name()} {cmb:22s} {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)
