"""Block-0 timeline of a split-K launch (PDL_TRACE build): where the per-unit time goes.
usage: PDL_LIB=build/libpdl_trace.so python scripts/probe_split_trace.py LAYER N SPLIT..."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W
L = _lib.lib()
L.pdl_debug_set_trace.argtypes = [ctypes.c_void_p]
N_EV, TN = 11, 4096
names = ["P_ISSUE", "S_FULL", "S_TFREE", "S_DONE", "M_READY", "M_ISSUED", "E_FULL", "E_DRAINED", "E_STORED", "M_WAITED", "M_LOOP"]
l = W.LAYERS[int(sys.argv[1]) - 1]
n = int(sys.argv[2])
x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
b = torch.rand(l.K, device='cuda')
pw = P.prepack_weights(w, channels=l.C)
y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
for s in [int(a) for a in sys.argv[3:]]:
    run = lambda: P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y, cfg={"split_k": s})
    for _ in range(2):
        run()
    tb = torch.zeros(N_EV * TN, dtype=torch.int64, device='cuda')
    L.pdl_debug_set_trace(ctypes.c_void_p(tb.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record()
    torch.cuda.synchronize()
    L.pdl_debug_set_trace(None)
    t = tb.cpu().numpy().reshape(N_EV, TN).astype(np.int64)
    t0 = t[t > 0].min()
    print(f"== {l.name()} n={n} split={s}: {e0.elapsed_time(e1)*1e3:.1f} us")
    st = t[8]
    for jt in range(8):
        v = st[1000 + jt * 8: 1000 + jt * 8 + 5]
        if v[0] > 0:
            dr = t[7][jt] - t0 if t[7][jt] > 0 else -1
            print(f"  unit {jt}: drained {dr} partial-written {v[0]-t0} fence+bar {v[1]-v[0]} "
                  f"wait {v[2]-v[1] if v[2] > 0 else -1} reduce {v[3]-v[2] if v[3] > 0 and v[2] > 0 else -1} "
                  f"stored {st[jt]-t0 if st[jt] > 0 else -1}")
    for i, nm in enumerate(names):
        v = t[i][:1000][t[i][:1000] > 0] - t0
        if len(v):
            print(f"  {nm:10s} n={len(v):3d} first={v.min():8d} last={v.max():8d}  " +
                  " ".join(str(int(a)) for a in np.sort(v)[:12]))
