"""Small per-GPU batches (the 8-GPU strong-scaling shard): host launch cost per
conv call, eager step vs CUDA-graph step, and per-layer device time from
graph replays of one layer (no host gaps)."""
import json
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

out = {}
for n in [int(a) for a in (sys.argv[1:] or ["32", "256"])]:
    bufs = []
    for l in W.LAYERS:
        x = torch.rand((n, l.C_alloc // 16, l.H, l.W, 16), device='cuda')
        w = torch.rand((l.K // 16, l.C_alloc // 16, l.R, l.S, 16, 16), device='cuda')
        b = torch.rand(l.K, device='cuda')
        pw = P.prepack_weights(w, channels=l.C)
        y = torch.empty((n, l.K // 16, l.P, l.Q, 16), device='cuda')
        bufs.append((l, x, pw, b, y))

    def call(i):
        l, x, pw, b, y = bufs[i]
        P.conv2d_nchw16c(x, pw, b, stride=l.stride, pad=l.pad, relu=True, out=y)

    def step():
        for i in range(len(bufs)):
            call(i)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    # host cost per call (GPU runs behind; 200 calls fit in the launch queue)
    t0 = time.perf_counter()
    for _ in range(10):
        step()
    host_us = (time.perf_counter() - t0) / (10 * len(bufs)) * 1e6
    torch.cuda.synchronize()

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    eager = timed(step, 20)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    graph = timed(g.replay, 20)
    per_layer = []
    for i, (l, *_r) in enumerate(bufs):
        gl = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gl, stream=s):
                for _ in range(10):
                    call(i)
        torch.cuda.synchronize()
        gl.replay()
        torch.cuda.synchronize()
        ms = timed(gl.replay, 5) / 10
        per_layer.append((l.name(), round(ms * 1e3, 1)))
    flops = sum(l.flops(n) for l in W.LAYERS)
    out[n] = {"host_us_per_call": round(host_us, 1), "eager_ms": round(eager, 4),
              "graph_ms": round(graph, 4), "eager_tflops": round(flops / eager / 1e9, 1),
              "graph_tflops": round(flops / graph / 1e9, 1),
              "sum_isolated_ms": round(sum(v for _, v in per_layer) / 1e3, 4),
              "per_layer_us_isolated_back_to_back": per_layer}
    print(json.dumps({n: out[n]}), flush=True)
    del bufs
    torch.cuda.empty_cache()
