"""Time explicit conv tile boxes (PDL_RASTER_TILE) against the library's pick, per layer.
    python scripts/probe_tile_shapes.py [N] [mode]"""
import sys
sys.path.insert(0, '.')
import torch
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import _lib, workloads as W

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mode = sys.argv[2] if len(sys.argv) > 2 else "3xtf32"
SHAPES = {
    3: [(8, 8, 2), (16, 8, 1), (14, 3, 3), (56, 2, 1), (28, 4, 1), (14, 9, 1)],
    6: [(14, 1, 9), (4, 4, 8), (7, 2, 9), (28, 1, 4), (28, 4, 1), (14, 3, 3)],
    7: [(14, 3, 3), (28, 4, 1), (7, 4, 4), (7, 6, 3), (4, 4, 8), (14, 1, 9)],
    8: [(14, 1, 9), (4, 4, 8), (28, 1, 4), (28, 4, 1), (7, 2, 9)],
    9: [(14, 1, 9), (4, 4, 8), (7, 2, 9), (28, 4, 1)],
    10: [(14, 1, 9), (4, 4, 8), (28, 1, 4), (28, 4, 1)],
    11: [(14, 1, 9), (14, 3, 3), (7, 2, 9), (14, 9, 1)],
    12: [(14, 3, 3), (14, 2, 4), (7, 6, 3), (14, 9, 1), (14, 1, 9), (7, 2, 9)],
    13: [(14, 1, 9), (14, 3, 3), (7, 2, 9), (14, 9, 1)],
    14: [(14, 1, 9), (14, 3, 3), (7, 2, 9)],
    15: [(14, 1, 9), (14, 3, 3), (14, 9, 1)],
    16: [(7, 1, 18), (7, 2, 9), (7, 7, 2), (4, 1, 32)],
    17: [(7, 7, 2), (7, 1, 18), (7, 2, 9), (7, 2, 7), (7, 4, 4)],
    18: [(7, 1, 18), (7, 7, 2), (7, 2, 9)],
    19: [(7, 1, 18), (7, 2, 9), (7, 7, 2)],
    20: [(7, 1, 18), (7, 7, 2), (7, 2, 9)],
}
flush = torch.empty(64 << 20, device='cuda')


def timeit(run, reps=15):
    ts = []
    for i in range(reps + 3):
        flush.add_(1.0)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); e.record(); e.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


for idx, shapes in SHAPES.items():
    l = W.LAYERS[idx - 1]
    x = torch.rand((N, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
    w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
    b = torch.rand(l.K, device='cuda')
    pw = P.prepack_weights(w, mode=mode, channels=l.C)
    y = torch.empty((N, l.K // 16, l.P, l.Q, 16), device='cuda')
    kw = dict(stride=l.stride, pad=l.pad, relu=True, mode=mode, out=y)
    res = []
    for name, cfg in [("auto", None), ("single", {"raster": 8}), ("seg", {"raster": 4})] + \
            [("%dx%dx%d" % s, {"raster": s[0] << 8 | s[1] << 16 | s[2] << 24}) for s in shapes if s[2] <= N]:
        try:
            sc = _lib.conv_schedule(N, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, _lib.MODES[mode], cfg=cfg)
            t = timeit(lambda: P.conv2d_nchw16c(x, pw, b, cfg=cfg, **kw))
            res.append((name, t, sc))
        except Exception as e:  # noqa: BLE001
            res.append((name, float('nan'), {"err": str(e)[:60]}))
    print(l.name(), f"N={N} {mode}")
    for name, t, sc in res:
        if "err" in sc:
            print(f"    {name:10s} ERR {sc['err']}")
        else:
            print(f"    {name:10s} {t:8.1f} us  tile {sc['tile_w']}x{sc['tile_h']}x{sc['tile_images']} m_tiles {sc['m_tiles']} "
                  f"split {sc['split']} halo {sc['halo']} seg {sc['seg_rows']} flat {sc['flat']} res {sc['resident']} bn {sc['bn']}", flush=True)
    del x, y
