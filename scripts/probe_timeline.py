"""Whole-kernel timeline of block 0 for small launches (PDL_TRACE build): where the fixed
cost of a short kernel goes (prologue, first load, k-loop, split-K exchange, stores, teardown).
    PDL_LIB=.../libpdl_trace.so python scripts/probe_timeline.py N idx [idx ...] | gM,N,K"""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W
L = _lib.lib()
L.pdl_debug_set_trace.argtypes = [ctypes.c_void_p]
N_EV, TN = 13, 4096
names = ["P_ISSUE", "S_FULL", "S_TFREE", "S_DONE", "M_READY", "M_ISSUED", "E_FULL", "E_DRAINED", "E_STORED",
         "M_WAITED", "M_LOOP", "KERNEL", "SPLIT"]
n = int(sys.argv[1])
for arg in sys.argv[2:]:
    if arg.startswith("g"):
        m, nn, k = (int(v) for v in arg[1:].split(","))
        a = torch.rand(m, k, device='cuda'); bm = torch.rand(k, nn, device='cuda'); c = torch.empty(m, nn, device='cuda')
        run = lambda: P.gemm(a, bm, c)
        name = f"gemm {m}x{nn}x{k}"
    else:
        l = W.PR1 if arg == "pr1" else W.LAYERS[int(arg) - 1]
        nb = 1 if arg == "pr1" else n
        x = torch.rand((nb, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
        w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
        b = torch.rand(l.K, device='cuda')
        pw = P.prepack_weights(w, channels=l.C)
        y = torch.empty((nb, l.K // 16, l.P, l.Q, 16), device='cuda')
        run = lambda: P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y)
        name = f"{l.name()} N={nb}"
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    flush = torch.empty(64 << 20, device='cuda'); flush.add_(1.0)
    tb = torch.zeros(N_EV * TN, dtype=torch.int64, device='cuda')
    L.pdl_debug_set_trace(ctypes.c_void_p(tb.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    L.pdl_debug_set_trace(None)
    t = tb.cpu().numpy().reshape(N_EV, TN).astype(np.int64)
    ev = {nm: t[i] for i, nm in enumerate(names)}
    k0 = ev["KERNEL"][0]
    rel = lambda v: int(v - k0) if v > 0 else -1
    def last(nm):
        v = ev[nm][ev[nm] > 0]
        return rel(v.max()) if len(v) else -1
    def first(nm):
        v = ev[nm][ev[nm] > 0]
        return rel(v.min()) if len(v) else -1
    nkb = int((ev["M_ISSUED"] > 0).sum())
    print(f"{name}: event-timed {e0.elapsed_time(e1)*1e3:.1f} us (cold L2); block 0 cycles from kernel entry:")
    print(f"   prologue done {rel(ev['KERNEL'][1])}, griddep wait done {rel(ev['KERNEL'][2])}, producer: entered {rel(ev['KERNEL'][5])} / "
          f"first tile decoded {rel(ev['KERNEL'][6])} / before first stage wait {rel(ev['KERNEL'][7])}, first TMA issue {first('P_ISSUE')}, "
          f"first stage landed {first('S_FULL')}, first MMA ready {first('M_READY')}, last MMA issued {last('M_ISSUED')} ({nkb} k-blocks), "
          f"first acc full {first('E_FULL')}, last drained {last('E_DRAINED')}, split bumped {first('SPLIT')}..{last('SPLIT')}, "
          f"last stored {last('E_STORED')}, epilogue exit {rel(ev['KERNEL'][3])}, dealloc {rel(ev['KERNEL'][4])}", flush=True)
