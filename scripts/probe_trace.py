"""Timeline of one CTA (block 0) through the tile engine (PDL_TRACE build)."""
import ctypes, json, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W
L = _lib.lib()
L.pdl_debug_set_trace.argtypes = [ctypes.c_void_p]
N_EV, TN = 13, 4096
names = ["P_ISSUE", "S_FULL", "S_TFREE", "S_DONE", "M_READY", "M_ISSUED", "E_FULL", "E_DRAINED", "E_STORED", "M_WAITED", "M_LOOP", "KERNEL", "SPLIT"]
out = {}
import os
CL = int(os.environ.get("CL", "0"))
cfg = {"cluster_m": CL} if CL else None
if os.environ.get("PAIR"):
    cfg = {"cluster_n": 2}
class _G:
    def __init__(self, m): self.m = m
    def name(self): return f"gemm{self.m}"
for arg in (sys.argv[1:] or ["3", "7", "4", "17"]):
    if arg.startswith("g"):
        m = int(arg[1:])
        l = _G(m)
        a = torch.rand(m, m, device='cuda'); bm = torch.rand(m, m, device='cuda'); c = torch.empty(m, m, device='cuda')
        run = lambda: P.gemm(a, bm, c, cfg=cfg)
    else:
        l = W.LAYERS[int(arg) - 1]
        n = int(os.environ.get("N", "256"))
        x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
        w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
        b = torch.rand(l.K, device='cuda')
        pw = P.prepack_weights(w, channels=l.C)
        y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
        run = lambda: P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y, cfg=cfg)
    for _ in range(2):
        run()
    tb = torch.zeros(N_EV * TN, dtype=torch.int64, device='cuda')
    L.pdl_debug_set_trace(ctypes.c_void_p(tb.data_ptr()))
    run()
    torch.cuda.synchronize()
    L.pdl_debug_set_trace(None)
    t = tb.cpu().numpy().reshape(N_EV, TN).astype(np.int64)
    t0 = t[t > 0].min()
    d = {nm: [int(v - t0) if v > 0 else -1 for v in t[i]] for i, nm in enumerate(names)}
    out[l.name()] = d
    nk = int((t[3] > 0).sum())  # k-blocks staged (S_DONE); the stem has no producer loads
    def col(nm): return np.array(d[nm][:nk], dtype=np.int64)
    mr, mi, sf, sd, stf, pi = col("M_READY"), col("M_ISSUED"), col("S_FULL"), col("S_DONE"), col("S_TFREE"), col("P_ISSUE")
    total = int(mi[nk - 1])
    print(f"  staging: S_FULL->S_TFREE median {np.median(stf - sf):.0f}, S_TFREE->S_DONE {np.median(sd - stf):.0f}, "
          f"S_DONE->next S_FULL {np.median(sf[1:] - sd[:-1]):.0f}; per-kb S_DONE spacing {np.median(np.diff(sd)):.0f}")
    ef, ed, es = (np.array([v for v in d[nm] if v >= 0], dtype=np.int64) for nm in ("E_FULL", "E_DRAINED", "E_STORED"))
    if len(es) > 2:
        print(f"  epilogue: full->drained median {np.median(ed[:len(ef)] - ef[:len(ed)]):.0f}, tiles {len(es)}, "
              f"store spacing {np.median(np.diff(es)):.0f}")
        nseg = max(1, len(ed) // max(1, len(es)))
        if nseg == 1 and len(ed) >= len(es):
            st = es[:len(ed)] - ed[:len(es)]
            wait_next = ef[1:len(es)] - es[:len(ef) - 1]
            print(f"  epilogue: drained->stored median {np.median(st):.0f}, stored->next full median "
                  f"{np.median(wait_next):.0f}")
    mma_wait = int(np.sum(np.maximum(mr[1:] - mi[:-1], 0)))
    gap = np.median(mr[1:] - mi[:-1])
    ml, mw = col("M_LOOP"), col("M_WAITED")
    print(f"CL={CL} median MMA gap issued->next ready {gap:.0f}: issued->loop {np.median(ml[1:]-mi[:-1]):.0f}, loop->waited {np.median(mw-ml):.0f}, waited->ready(fence) {np.median(mr-mw):.0f}")
    print(f"{l.name()}: kblocks {nk}, span {total} cyc ({total/nk:.0f}/kb); MMA waiting for staging {mma_wait/total:.1%}; "
          f"median TMA latency (issue->full) {np.median(sf - pi):.0f}; staging busy full->done median {np.median(sd - sf):.0f}; "
          f"tfree wait median {np.median(stf - sf):.0f}; MMA issue median {np.median(mi - mr):.0f}", flush=True)
json.dump(out, open("gpurun_out/trace.json", "w"))
