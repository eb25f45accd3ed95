"""ResNet layer 3 (64 -> 64, 3x3, 56x56) schedules, isolated graph replay at 256 images."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

for idx in [int(a) for a in sys.argv[1:] if a.isdigit()] or [3]:
    l = W.LAYERS[idx - 1]
    n = 256
    x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    mode = "tf32" if "--tf32" in sys.argv else "3xtf32"
    pw = P.prepack_weights(w, channels=l.C, mode=mode)
    y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
    mode = "tf32" if "--tf32" in sys.argv else "3xtf32"
    menu = [("default", None), ("no_halo", {"raster": 16})]
    if mode == "tf32" and l.K >= 128:
        menu += [("bk64", {"bk": 64}), ("bk32", {"bk": 32})]
    if mode == "tf32" and l.K % 256 == 0:
        menu += [("bn256_no_halo", {"bn": 256, "bk": 32, "raster": 16}), ("bk32_no_halo", {"bk": 32, "raster": 16})]
    elif mode == "3xtf32" and l.K >= 128:
        menu += [("bk64", {"bk": 64})]
    if "--pairs" in sys.argv:
        menu += [("pair", {"cluster_n": 2}), ("cl2", {"cluster_m": 2})]
    if l.K == 64:
        menu += [("halo_cg4", {"raster": 64}), ("bk32", {"bk": 32}), ("bk32_no_halo", {"bk": 32, "raster": 16})]
    for name, cfg in menu:
        def call():
            P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y, cfg=cfg, mode=mode)
        try:
            call()
        except Exception as e:
            print(name, "error", e)
            continue
        torch.cuda.synchronize()
        if cfg is None:
            y_ref = y.clone()
        else:
            err = float((y - y_ref).abs().max() / y_ref.abs().max())
            print(f"  {name}: rel diff vs default {err:.2e}")
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(5):
                    call()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"{l.name()} {name}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
