"""Where do wrong halo + split-K results land?  Repeats a failing config and maps the
wrong outputs onto tiles / channel blocks / pixels."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P  # noqa: E402
from paper_2006_02230_b200 import workloads as W  # noqa: E402

cases = [("pr1", W.PR1, 1, "3xtf32", {"bk": 32, "split_k": 18}),
         ("L17", W.LAYERS[16], 32, "tf32", {"split_k": 4}),
         ("L12", W.LAYERS[11], 8, "3xtf32", {"split_k": 16})]
for name, l, n, mode, cfg in cases:
    torch.manual_seed(0)
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda') * 2 - 1
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda') * 2 - 1
    pw = P.prepack_weights(w, channels=l.C, mode=mode)
    base = P.conv2d_nchw16c(x, pw, stride=l.stride, pad=l.pad, mode=mode, cfg={"split_k": 1, "bk": cfg.get("bk", 0)})
    tol = 1e-5 if mode == "3xtf32" else 1e-3
    for rep in range(4):
        y = P.conv2d_nchw16c(x, pw, stride=l.stride, pad=l.pad, mode=mode, cfg=cfg)
        torch.cuda.synchronize()
        d = (y - base).abs()
        scale = base.abs().max()
        bad = d > tol * scale
        nb = int(bad.sum())
        msg = f"{name} rep {rep}: max-rel {float(d.max() / scale):.2e}, {nb} wrong of {bad.numel()}"
        if nb:
            idx = bad.nonzero()
            imgs = sorted(set(idx[:, 0].tolist()))[:8]
            kts = sorted(set(idx[:, 1].tolist()))
            ps = sorted(set(idx[:, 2].tolist()))
            qs = sorted(set(idx[:, 3].tolist()))
            # per (img, kt) plane: fraction wrong
            planes = bad.any(dim=-1).float().mean(dim=(2, 3))
            full = int((planes > 0.99).sum())
            msg += f"\n   imgs {imgs} kts {kts}\n   rows {ps[:20]} cols {qs[:20]}\n   planes fully wrong {full}, " \
                   f"partial {int(((planes > 0) & (planes <= 0.99)).sum())}"
            # relative size of the error vs one tap's contribution
            ratio = float((d[bad] / base.abs()[bad].clamp_min(1e-3)).median())
            msg += f"; median |err|/|y| {ratio:.2f}"
        print(msg, flush=True)
