#!/usr/bin/env python
"""Measure every legal tile variant of every ResNet-50 layer on the B200.

For each layer and mode: check each variant against the library default
(bitwise, N=2), then time it fused (bias+ReLU) at the bench batch with CUDA
events, L2 flushed between repetitions.  Writes one JSON document with, per
variant, the measured time, the pipeline-model prediction, the Eq. 1 cost and
the per-level working-set statistics -- the data `scripts/fit_ranker.py` fits
the pipeline model and trains the DNN judge on.

    python scripts/sweep_variants.py --out gpurun_out/sweep.json [--batch 256]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2006_02230_b200 import ops, rank, variants, workloads  # noqa: E402
from paper_2006_02230_b200.machine import default_machine  # noqa: E402


def time_variant(layer, X, PW, B, cfg, mode, reps, flush):
    out = torch.empty(X.shape[0], layer.K // 16, layer.P, layer.Q, 16, device="cuda")
    run = lambda: ops.conv2d_nchw16c(X, PW, B, stride=layer.stride, pad=layer.pad, relu=True,
                                     mode=mode, channels=layer.C, cfg=cfg, out=out)
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.add_(1.0)
        torch.cuda._sleep(20000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--modes", default="3xtf32,tf32")
    ap.add_argument("--layers", default="")
    ap.add_argument("--cap", type=int, default=256, help="variants per layer and mode")
    args = ap.parse_args()
    torch.manual_seed(0)
    m = default_machine()
    pm = rank.PipelineModel.load()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    layers = workloads.resnet50_v1_layers()
    if args.layers:
        keep = {int(t) for t in args.layers.split(",")}
        layers = [L for L in layers if L.idx in keep]
    doc = {"batch": args.batch, "device": torch.cuda.get_device_name(), "layers": []}
    t0 = time.time()
    for L in layers:
        n = args.batch
        X = torch.rand(n, L.C_alloc // 16, L.H, L.W, 16, device="cuda") * 2 - 1
        if L.C != L.C_alloc:
            X[:, :, :, :, L.C:] = 0
        x2, w, b = workloads.conv_inputs(L, 2, seed=L.idx)
        Wt, Bt = torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda()
        X2 = torch.from_numpy(x2).cuda()
        for mode in args.modes.split(","):
            PW = ops.prepack_weights(Wt, mode, channels=L.C)
            ref = ops.conv2d_nchw16c(X2, PW, Bt, stride=L.stride, pad=L.pad, relu=True,
                                     mode=mode, channels=L.C)
            vs = variants.generate_variants(L, variants.VariantConfig(modes=(mode,), cap=args.cap), n_images=n)
            rows = {}
            for v in vs:
                cfg = variants.emit_launch(v)
                got = ops.conv2d_nchw16c(X2, PW, Bt, stride=L.stride, pad=L.pad, relu=True,
                                         mode=mode, channels=L.C, cfg=cfg)
                bitwise = bool(torch.equal(got, ref))
                rel = float((got - ref).abs().max()) / (float(ref.abs().max()) or 1.0)
                legal = rel <= variants.MODE_TOLERANCE[mode]
                med, best = time_variant(L, X, PW, Bt, cfg, mode, args.reps, flush)
                st = rank.stats_for_variant(L, v, n, m)
                rows[v.vid] = {**v.provenance(), "legal": legal, "bitwise": bitwise, "max_rel": rel,
                               "schedule": variants.schedule(L, v, n),
                               "ms": med, "ms_min": best,
                               "tflops": L.flops(n) / (med * 1e-3) / 1e12,
                               "model_ms": pm.predict_seconds(L, v, n) * 1e3,
                               "cost": float(rank.cost_of_stats(st, m)),
                               "stats": [st.ws_l1, st.ws_l2, st.ws_l3, st.ws_mem]}
            med, best = time_variant(L, X, PW, Bt, None, mode, args.reps, flush)
            doc["layers"].append({"layer": L.name(), "idx": L.idx, "mode": mode, "batch": n,
                                  "C": L.C, "K": L.K, "H": L.H, "R": L.R, "stride": L.stride,
                                  "flops": L.flops(n), "default_ms": med, "variants": rows})
            order = sorted(rows, key=lambda k: rows[k]["ms"])
            print(f"{L.name()} {mode}: default {med:.4f} ms; best {order[0]} "
                  f"{rows[order[0]]['ms']:.4f} ms; worst {order[-1]} {rows[order[-1]]['ms']:.4f}; "
                  f"illegal {[k for k in rows if not rows[k]['legal']]}", flush=True)
        del X
        torch.cuda.empty_cache()
    doc["elapsed_s"] = time.time() - t0
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
