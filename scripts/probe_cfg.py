"""Time layers under the default schedule and under tile-config overrides (isolated, L2 flushed).
    [PDL_LIB=...] python scripts/probe_cfg.py N mode '{"bk": 64}' idx [idx ...]"""
import json, sys
sys.path.insert(0, '.')
import torch
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W

N = int(sys.argv[1]); mode = sys.argv[2]; cfgs = [None] + [json.loads(c) for c in sys.argv[3].split(";")]
flush = torch.empty(64 << 20, device='cuda')
for idx in [int(a) for a in sys.argv[4:]]:
    l = W.LAYERS[idx - 1]
    x = torch.rand((N, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, mode=mode, channels=l.C)
    y = torch.empty((N, l.K // 16, l.P, l.Q, 16), device='cuda')
    ref = None
    out = []
    for cfg in cfgs:
        try:
            run = lambda: P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, mode=mode, out=y, cfg=cfg)
            for _ in range(3):
                run()
            ts = []
            for i in range(11):
                flush.add_(1.0)
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); run(); e.record(); e.synchronize()
                ts.append(a.elapsed_time(e))
            ts.sort()
            if ref is None:
                ref = y.clone()
                err = 0.0
            else:
                err = float((y - ref).abs().max() / ref.abs().max())
            sc = _lib.conv_schedule(N, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, _lib.MODES[mode], cfg=cfg)
            out.append(f"{json.dumps(cfg)}: {ts[5]*1e3:.1f} us (bn {sc['bn']} bk {sc['bk']} split {sc['split']} halo {sc['halo']} rel {err:.1e})")
        except Exception as ex:  # noqa: BLE001
            out.append(f"{json.dumps(cfg)}: ERR {str(ex)[:80]}")
    print(l.name(), f"N={N} {mode}:", " | ".join(out), flush=True)
