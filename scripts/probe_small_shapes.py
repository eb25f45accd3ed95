"""Small-shape schedules (PR1, small / rectangular GEMMs, 32-image layers): per-launch
time of back-to-back launches over rotated inputs for a menu of tile configs.

    python scripts/probe_small_shapes.py [pr1] [gemm] [layers 6 16 20 ...]
"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P  # noqa: E402
from paper_2006_02230_b200 import workloads as W  # noqa: E402


def bench(calls, reps=3):
    for c in calls:
        c()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for c in calls:
                c()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / len(calls) * 1e3  # us per launch


def conv_menu(layer, n, mode, menu, nrot):
    x = torch.rand((n, layer.C_alloc // 16, layer.H, layer.W, 16), device='cuda') * 2 - 1
    w = torch.rand((layer.K // 16, layer.C_alloc // 16, layer.R, layer.S, 16, 16), device='cuda') * 2 - 1
    b = torch.rand(layer.K, device='cuda') - 0.5
    pw = P.prepack_weights(w, channels=layer.C, mode=mode)
    xs = [x.clone() for _ in range(nrot)]
    ys = [torch.empty((n, layer.K // 16, layer.P, layer.Q, 16), device='cuda') for _ in range(nrot)]
    ref = None
    for name, cfg in menu:
        calls = [lambda i=i, cfg=cfg: P.conv2d_nchw16c(xs[i], pw, b, stride=layer.stride, pad=layer.pad,
                                                       relu=True, mode=mode, out=ys[i], cfg=cfg)
                 for i in range(nrot)]
        try:
            calls[0]()
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(f"  {layer.name()} n={n} {mode} {name}: error {e}")
            continue
        if ref is None:
            ref = ys[0].clone()
        diff = float((ys[0] - ref).abs().max() / ref.abs().max())
        us = bench(calls)
        print(f"  {layer.name()} n={n} {mode} {name}: {us:.2f} us/launch (rel diff {diff:.1e})", flush=True)


def gemm_menu(m, n, k, mode, menu):
    nset = max(8, min(256, (320 << 20) // (4 * (m * k + k * n + m * n))))
    sets = [(torch.rand((m, k), device='cuda') * 2 - 1, torch.rand((k, n), device='cuda') * 2 - 1,
             torch.empty((m, n), device='cuda')) for _ in range(nset)]
    for name, cfg in menu:
        calls = [lambda s=s, cfg=cfg: P.gemm(s[0], s[1], s[2], mode=mode, cfg=cfg) for s in sets]
        try:
            calls[0]()
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(f"  gemm {m}x{n}x{k} {mode} {name}: error {e}")
            continue
        us = bench(calls)
        print(f"  gemm {m}x{n}x{k} {mode} {name}: {us:.2f} us/launch ({2*m*n*k/us/1e6:.1f} TF/s)", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    modes = ["3xtf32", "tf32"] if "--tf32" in args else ["3xtf32"]
    if "pr1" in args:
        for mode in modes:
            menu = [("default", None), ("split3", {"split_k": 3}), ("split9", {"split_k": 9}),
                    ("bk32", {"bk": 32}), ("bk32_split3", {"bk": 32, "split_k": 3}),
                    ("bk32_split6", {"bk": 32, "split_k": 6}), ("bk32_split9", {"bk": 32, "split_k": 9}),
                    ("bk32_split18", {"bk": 32, "split_k": 18}), ("nohalo_split9", {"split_k": 9, "raster": 16})]
            conv_menu(W.PR1, 1, mode, menu, 200)
    if "gemm" in args:
        for mode in modes:
            for (m, n, k) in [(64, 64, 64), (256, 256, 256), (512, 512, 512), (1024, 1024, 1024),
                              (3136, 64, 576), (784, 512, 128), (49, 2048, 512)]:
                menu = [("default", None), ("bn64", {"bn": 64}), ("split2", {"split_k": 2}),
                        ("split4", {"split_k": 4}), ("split8", {"split_k": 8}), ("bn64_split4", {"bn": 64, "split_k": 4})]
                gemm_menu(m, n, k, mode, menu)
    if "layers" in args:
        idx = [int(a) for a in args[args.index("layers") + 1:] if a.isdigit()]
        for mode in modes:
            for i in idx:
                l = W.LAYERS[i - 1]
                menu = [("default", None), ("split1", {"split_k": 1}), ("split2", {"split_k": 2}),
                        ("split4", {"split_k": 4}), ("bn64", {"bn": 64}), ("bn64_split2", {"bn": 64, "split_k": 2})]
                conv_menu(l, 32, mode, menu, 4)
