"""Forced split-K sweep: every split factor on a few conv shapes / modes / halo on-off,
compared with the unsplit result (max-rel), to localise wrong split-K results."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P  # noqa: E402
from paper_2006_02230_b200 import workloads as W  # noqa: E402

CASES = [("pr1", W.PR1, 1), ("L17", W.LAYERS[16], 32), ("L12", W.LAYERS[11], 8), ("L03", W.LAYERS[2], 2),
         ("L20", W.LAYERS[19], 32)]
for name, l, n in CASES:
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda') * 2 - 1
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda') * 2 - 1
    b = torch.rand(l.K, device='cuda') - 0.5
    for mode in ("3xtf32", "tf32"):
        pw = P.prepack_weights(w, channels=l.C, mode=mode)
        for extra in ({}, {"bk": 32}, {"raster": 16}, {"bk": 32, "raster": 16}):
            try:
                base = P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, mode=mode,
                                        cfg=dict(extra, split_k=1))
            except Exception as e:  # noqa: BLE001
                print(name, mode, extra, "base error", e)
                continue
            bad = []
            for s in range(2, 25):
                try:
                    y = P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, mode=mode,
                                         cfg=dict(extra, split_k=s))
                except Exception as e:  # noqa: BLE001
                    bad.append((s, "err"))
                    continue
                torch.cuda.synchronize()
                d = float((y - base).abs().max() / base.abs().max())
                if d > (1e-5 if mode == "3xtf32" else 1e-3):
                    bad.append((s, f"{d:.1e}"))
            print(f"{name} n={n} {mode} {extra}: bad splits {bad}", flush=True)
