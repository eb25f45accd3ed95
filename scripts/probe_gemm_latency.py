"""Per-launch time of small GEMMs (graph-replayed, warm L2) vs cluster size, and a
trivial library kernel for the launch floor."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P


def per_launch(fn, n=50):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * n) * 1e3


y = torch.zeros(1, 1, 1, 4, 16, device="cuda")
print(f"bias_relu on 64 floats: {per_launch(lambda: P.bias_relu_(y, None)):.2f} us", flush=True)
for m in (64, 256, 512, 1024, 2048):
    a = torch.rand(m, m, device="cuda")
    b = torch.rand(m, m, device="cuda")
    c = torch.empty(m, m, device="cuda")
    res = []
    for name, cfg in (("default", None), ("cl1", {"cluster_m": 1}), ("cl1_nosplit", {"cluster_m": 1, "split_k": 1}),
                      ("bn64_cl1", {"cluster_m": 1, "bn": 64}), ("fp32simt", "simt")):
        if cfg == "simt":
            fn = lambda: P.gemm(a, b, c, mode="fp32")
        else:
            fn = lambda cfg=cfg: P.gemm(a, b, c, cfg=cfg)
        res.append(f"{name}={per_launch(fn):.2f}us")
    print(f"gemm {m}^3: " + " ".join(res), flush=True)
