#!/usr/bin/env python
"""bench.py -- B200 benchmark of the PolyDL hot path (driver contract).

Default workload (BASELINE.json configs[3]/[4]): one "step" = one forward pass
of the 20 distinct ResNet-50 v1 conv layers, each a FUSED conv + bias + ReLU in
3xTF32 (fp32-accurate), nChw16c / KCRS16c16k, on a global minibatch of 256
images sharded contiguously across the ranks (256/G per GPU, no collective on
the path; weights replicated once with an NCCL broadcast before timing).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload suite|gemm|pr1] [--mode 3xtf32|tf32] [--unfused]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv/GEMM GFLOP/s per layer and % of B200 roofline at 1/2/4/8 GPUs vs CPU oracle"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs of this node; > 1 without torchrun re-launches this script "
                         "under torch.distributed.run with one rank per GPU")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="suite", choices=["suite", "gemm", "pr1", "layout"])
    ap.add_argument("--mode", default="3xtf32", choices=["3xtf32", "tf32"])
    ap.add_argument("--batch", type=int, default=256, help="global minibatch (suite)")
    ap.add_argument("--unfused", action="store_true", help="also time conv + separate bias/ReLU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the sub-objects for the other BASELINE configs (gemm, pr1, n28, tf32)")
    ap.add_argument("--box-tiles", action="store_true", help="A/B: disable segment tiles (PDL_RASTER_BOX_TILES)")
    ap.add_argument("--m-fastest", action="store_true", help="A/B: output-pixel tiles fastest (PDL_RASTER_M_FASTEST)")
    ap.add_argument("--single-image-tiles", action="store_true",
                    help="A/B: round-1 tile geometry, no multi-image box search (PDL_RASTER_SINGLE_IMAGE_TILES)")
    ap.add_argument("--no-halo", action="store_true", help="A/B: per-tap A boxes for 3x3 layers (PDL_RASTER_NO_HALO)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA-graph replay of the step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="cpu_baseline sample budget")
    ap.add_argument("--cluster", type=int, default=0, help="override CTAs per weight-multicast cluster")
    ap.add_argument("--schedule", default="default", choices=["default", "ranked"],
                    help="tile config per layer: library default or the trained ranker's pick")
    return ap.parse_args()


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(gpus: int) -> None:
    """`python bench.py --gpus N` (N > 1, not already under torchrun): replace this
    process by torch.distributed.run with one rank per GPU of this node (NCCL over
    127.0.0.1); rank 0 prints the JSON line, the exit status is torchrun's."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            m = json.load(f)
        peaks.update(hbm_gbs=float(m["hbm_gbs"]), bf16_tflops=float(m["bf16_tflops"]),
                     bf16_tflops_sustained=float(m.get("bf16_tflops_sustained", m["bf16_tflops"])),
                     source="MEASURED_PEAKS.json")
    t = os.path.join(ROOT, "profiles", "peaks_tf32.json")
    if os.path.exists(t):
        with open(t) as f:
            peaks["cublas_tf32_tflops"] = float(json.load(f)["tf32_tflops"])
    return peaks


def mode_peak(peaks, mode: str):
    """(FLOP/s, label) of the tensor roofline of `mode`: the measured dense bf16
    burst rate / 2 (tcgen05 kind::tf32 runs at half the bf16 rate) and / 3 more
    for 3xTF32 (three tensor passes per fp32 product)."""
    div = 3.0 if mode == "3xtf32" else 1.0
    tf = peaks["bf16_tflops"] / 2.0 / div
    label = (f"{peaks['source']} bf16 dense burst {peaks['bf16_tflops']:.1f} TF/s / 2 (tf32)"
             + (" / 3 (3xTF32 = 3 tensor passes)" if mode == "3xtf32" else ""))
    return tf * 1e12, label


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s, p in zip(sm, power) if p > 200] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------------------- helpers
def ncu_traffic(kernel_tag: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        s = json.load(f)
    ent = s.get("kernels", {}).get(kernel_tag)
    return None if ent is None else ent.get("dram_bytes")


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_prepare(layers):
    import oracle
    from paper_2006_02230_b200 import workloads as W
    prepared = []
    for layer in layers:
        x, w, b = W.conv_inputs(layer, 1, seed=900 + layer.idx)
        xp = oracle.pad_nchw16c(x, layer.R, layer.S, layer.stride, layer.pad)
        y = np.empty((1, layer.K // 16, layer.P, layer.Q, 16), np.float32)
        prepared.append((layer, xp, np.ascontiguousarray(w), b, y))
    return prepared


def cpu_step(prepared, threads):
    import oracle
    for layer, xp, w, b, y in prepared:
        oracle.cpu_conv2d_f32(xp, w, b, layer.stride, layer.P, layer.Q, relu=True,
                              threads=threads, out=y)


def cpu_suite_sample(layers, seconds_budget: float, threads: int):
    """Time the oracle's fp32 Fig. 9 port (kind "port") on 1 image per layer,
    repeated up to the time budget.  Returns (GFLOP/s, reps, seconds)."""
    prepared = cpu_prepare(layers)
    flops = sum(l.flops(1) for l in layers)
    cpu_step(prepared, threads)  # page-in
    t_total, reps = 0.0, 0
    while reps == 0 or (t_total < seconds_budget and reps < 1000):
        t0 = time.perf_counter()
        cpu_step(prepared, threads)
        t_total += time.perf_counter() - t0
        reps += 1
    return flops * reps / t_total / 1e9, reps, t_total


def cpu_torch_onednn(layers, seconds_budget: float, threads: int):
    """The paper's comparison library (oneDNN) as bundled in torch:
    F.conv2d + bias + ReLU in NCHW fp32 on the host cores, 1 image per layer."""
    import torch
    import torch.nn.functional as F
    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(5)
    data = []
    for l in layers:
        x = torch.rand((1, l.C, l.H, l.W), generator=g) * 2 - 1
        w = torch.rand((l.K, l.C, l.R, l.S), generator=g) * 2 - 1
        b = torch.rand((l.K,), generator=g) - 0.5
        data.append((l, x, w, b))
    flops = sum(l.flops(1) for l in layers)

    def step():
        with torch.no_grad():
            for l, x, w, b in data:
                F.relu(F.conv2d(x, w, b, stride=l.stride, padding=l.pad))

    step()
    t_total, reps = 0.0, 0
    while reps == 0 or (t_total < seconds_budget and reps < 1000):
        t0 = time.perf_counter()
        step()
        t_total += time.perf_counter() - t0
        reps += 1
    return {"value": round(flops * reps / t_total / 1e9, 2), "unit": "GFLOP/s", "threads": threads,
            "library": f"torch {torch.__version__} CPU conv2d (oneDNN, mkldnn enabled="
                       f"{torch.backends.mkldnn.is_available()})",
            "sample": f"NCHW fp32, 1 image per layer x {len(layers)} layers, bias+ReLU, {reps} reps "
                      f"in {t_total:.1f} s"}


def reference_interpret_record(total_flops: float):
    """The reference's own CPU path (looprank.simcache.interpret) measured in the build
    container by scripts/time_interpret.py (it cannot run on the GPU box)."""
    p = os.path.join(ROOT, "profiles", "interpret_ref_r2.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        r = json.load(f)
    us = float(r["conv_us_per_mac_median"])
    return {"us_per_mac": us, "gflops": round(2.0 / (us * 1e-6) / 1e9, 6),
            "extrapolated_s_per_suite_step": round(total_flops / 2.0 * us * 1e-6, 1),
            "where": r["where"], "what": r["what"],
            "source": "profiles/interpret_ref_r2.json (measured, not timed in this run)"}


def time_calls(torch, calls, steps: int, stream, graph: bool = True, per_call: int = 0):
    """ms per pass over `calls` (a CUDA graph of one pass, replayed `steps` times;
    eager launches with graph=False) and, if per_call > 0, per-call ms from that
    many eager passes with device events around each call."""
    for c in calls:
        c()
    torch.cuda.synchronize()
    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                for c in calls:
                    c()
        stream.wait_stream(side)
        g.replay()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        if g is not None:
            g.replay()
        else:
            for c in calls:
                c()
    e1.record(stream)
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / steps
    per = []
    if per_call:
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in calls] for _ in range(per_call)]
        for r in range(per_call):
            for i, c in enumerate(calls):
                ev[r][i][0].record(stream)
                c()
                ev[r][i][1].record(stream)
        torch.cuda.synchronize()
        per = [sum(ev[r][i][0].elapsed_time(ev[r][i][1]) for r in range(per_call)) / per_call
               for i in range(len(calls))]
    return total, per


def layer_row(W, layer, n, ms, peak, hbm):
    rf = W.Roofline(layer.flops(n), layer.bytes(n, bias=True), peak, hbm)
    return {"layer": layer.name(), "ms": round(ms, 4),
            "gflops": round(layer.flops(n) / (ms / 1e3) / 1e9, 1),
            "bound": rf.bound, "roofline_frac": round(rf.fraction(ms / 1e3), 3)}


# ----------------------------------------------------------------------------- our arm
def run_suite(args, rank, world, local):
    import torch
    import torch.distributed as dist
    import paper_2006_02230_b200 as P
    from paper_2006_02230_b200 import _lib, workloads as W

    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} "
                         f"visible GPU(s)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if not P.device_ok():
        raise SystemExit("libpdl.so: no sm_100 device")
    from paper_2006_02230_b200.shard import max_over_ranks, replicate_, shard_images
    _, n_local = shard_images(args.batch, world, rank)
    if n_local == 0:
        raise SystemExit(f"--batch {args.batch} leaves rank {rank} of {world} without images")
    layers = W.LAYERS
    peaks = load_peaks()
    hbm = peaks["hbm_gbs"] * 1e9
    mpeak, mpeak_label = mode_peak(peaks, args.mode)

    # ---- data: inputs seeded per (layer, rank); weights from rank 0, broadcast once
    bufs = []
    for layer in layers:
        ca = layer.C_alloc
        g = torch.Generator(device=dev)
        g.manual_seed(10_000 * layer.idx + rank)
        x = torch.rand((n_local, ca // 16, layer.H, layer.W, 16), generator=g, device=dev) * 2 - 1
        gw = torch.Generator(device=dev)
        gw.manual_seed(7 + layer.idx)
        w = torch.rand((layer.K // 16, ca // 16, layer.R, layer.S, 16, 16), generator=gw,
                       device=dev) * 2 - 1
        b = torch.rand((layer.K,), generator=gw, device=dev) - 0.5
        if layer.C != ca:
            x[..., layer.C:] = 0
            w[:, :, :, :, layer.C:, :] = 0
        replicate_([w, b])
        pw = P.prepack_weights(w, mode=args.mode, channels=layer.C)
        y = torch.empty((n_local, layer.K // 16, layer.P, layer.Q, 16), device=dev)
        bufs.append((layer, x, w, b, pw, y))
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    launches_per_step = 0
    cfg = {"cluster_m": args.cluster} if args.cluster else None
    if args.box_tiles:  # A/B: no multi-image segment tiles
        cfg = dict(cfg or {}, raster=2)
    if args.m_fastest:  # A/B: tile-loop interchange (pixel tiles fastest)
        cfg = dict(cfg or {}, raster=(cfg or {}).get("raster", 0) | 1)
    if args.single_image_tiles:  # A/B: a tile holds several images only when a whole image fits
        cfg = dict(cfg or {}, raster=(cfg or {}).get("raster", 0) | 8)
    if args.no_halo:  # A/B: one A box per tap for 3x3 layers
        cfg = dict(cfg or {}, raster=(cfg or {}).get("raster", 0) | 16)
    if args.schedule == "ranked":
        from paper_2006_02230_b200 import rank as rk, variants
        cfgs = [variants.emit_launch(rk.choose_variant(l, n_local, args.mode)) for l in layers]
    else:
        cfgs = [cfg] * len(layers)

    def step(ev=None):
        nonlocal launches_per_step
        cnt = 0
        for i, (layer, x, w, b, pw, y) in enumerate(bufs):
            if ev is not None:
                ev[i][0].record(stream)
            P.conv2d_nchw16c(x, pw, b, stride=layer.stride, pad=layer.pad, relu=True,
                             mode=args.mode, out=y, cfg=cfgs[i])
            cnt += _lib.last_launch_count()
            if ev is not None:
                ev[i][1].record(stream)
        launches_per_step = cnt

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # The step's 20 launches are captured once in a CUDA graph and replayed: at
    # small per-GPU batches (32 images = the 8-GPU shard) a layer runs ~40 us,
    # about the host cost of two launches through Python, so eager launching
    # would time the host.  The graph replays the same kernels on the same
    # buffers; nothing is skipped.
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                step()
        stream.wait_stream(side)
        graph.replay()
        torch.cuda.synchronize()

    # ---- timed region (device time, max over ranks)
    clocks = ClockSampler(local)
    ev_layers = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in bufs] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before load starts
    t_start.record(stream)
    for k in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step(ev_layers[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = max_over_ranks(t_start.elapsed_time(t_end), dev)
    ms_step = ms / args.steps
    if graph is not None:
        # per-layer breakdown: a separate eager pass with device events around each launch
        for k in range(args.steps):
            step(ev_layers[k])
        torch.cuda.synchronize()
    total_flops = sum(l.flops(args.batch) for l in layers)
    value = total_flops / (ms_step / 1e3) / 1e9

    # ---- per-layer breakdown (this rank's device events)
    per_layer = []
    for i, (layer, *_rest) in enumerate(bufs):
        lms = sum(ev_layers[k][i][0].elapsed_time(ev_layers[k][i][1]) for k in range(args.steps)) / args.steps
        per_layer.append(dict(layer_row(W, layer, n_local, lms, mpeak, hbm), share=None))
    tot_layer_ms = sum(d["ms"] for d in per_layer)
    for d in per_layer:
        d["share"] = round(d["ms"] / tot_layer_ms, 3)

    # ---- dominant kernel roofline (contract object)
    dom_i = max(range(len(per_layer)), key=lambda i: per_layer[i]["ms"])
    dom_layer = bufs[dom_i][0]
    dom_s = per_layer[dom_i]["ms"] / 1e3
    rf = W.Roofline(dom_layer.flops(n_local), dom_layer.bytes(n_local, bias=True), mpeak, hbm)
    if rf.bound == "tensor":
        achieved = dom_layer.flops(n_local) / dom_s / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(mpeak / 1e12, 1),
                "unit": "TFLOP/s", "frac": round(achieved / (mpeak / 1e12), 4),
                "peak_source": mpeak_label + " (the kernel runs at burst clocks: see clocks)"}
        if "cublas_tf32_tflops" in peaks:
            ct = peaks["cublas_tf32_tflops"] / (3.0 if args.mode == "3xtf32" else 1.0)
            roof["frac_vs_cublas_tf32"] = round(achieved / ct, 4)
            roof["cublas_tf32_source"] = ("profiles/peaks_tf32.json: cuBLAS TF32 8192^3 on B200 "
                                          f"{peaks['cublas_tf32_tflops']:.1f} TF/s"
                                          + (" / 3" if args.mode == "3xtf32" else ""))
    else:
        achieved = dom_layer.bytes(n_local, bias=True) / dom_s / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "peak_source": peaks["source"]}
    roof.update(kernel=f"tile_mma_kernel[{dom_layer.name()}]",
                algorithmic_per_launch={"flops": dom_layer.flops(n_local),
                                        "bytes": dom_layer.bytes(n_local, bias=True)},
                avg_launch_ms=round(dom_s * 1e3, 4), traffic=ncu_traffic(dom_layer.name()))

    out = {"metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded U[-1,1) activations/weights, U[-0.5,0.5) bias; ResNet-50 "
                   "v1 shapes only, no dataset or checkpoint)",
           "config": {"workload": "resnet50_v1_20_distinct_layers_fused_conv_bias_relu",
                      "global_batch": args.batch, "per_gpu_batch": n_local, "mode": args.mode,
                      "layout": "nChw16c x / KCRS16c16k w (prepacked once) / nKhw16k y",
                      "parallelism": f"batch-sharded x{world}, no collective",
                      "schedule": args.schedule,
                      "launch": "eager" if args.no_graph else "cuda graph of the step's launches, replayed per step; per-layer ms from a separate eager pass with events",
                      "l2": "step working set %.1f GB >> 126 MB L2; each layer's inputs were "
                            "last touched one full step earlier" % (
                                sum(l.bytes(n_local) for l in layers) / 1e9),
                      "flops_per_step": total_flops},
           "roofline": roof, "clocks": clk, "gpu_launches": launches_per_step * args.steps,
           "layers": per_layer}

    # ---- e2e through the public API with host buffers
    if not args.no_e2e:
        out["e2e"] = run_suite_e2e(args, bufs, P, torch, dev, world, dist, total_flops, stream)
        # the same step with the stem's x in the compact [N][H][W][4] layout (PDL_X_NCHW4C):
        # reported beside the nChw16c headline, never instead of it
        out["e2e_compact_stem"] = run_suite_e2e(args, bufs, P, torch, dev, world, dist, total_flops,
                                                stream, compact_stem=True)
    if rank == 0 and world == 1 and not args.no_extras:
        out["stem_compact"] = run_stem_compact(args, bufs, P, W, torch, stream, peaks, per_layer)

    # ---- unfused GPU baseline comparison (optional)
    if args.unfused:
        out["unfused"] = run_unfused(args, bufs, P, torch, stream)

    # ---- the other BASELINE configs (single-GPU configs: rank 0 at N=1 only)
    if rank == 0 and world == 1 and not args.no_extras and args.schedule == "default" and cfg is None:
        out["n28"] = run_n28(args, bufs, P, W, torch, stream, peaks)
        if args.mode == "3xtf32" and args.batch == 256:
            out["tf32"] = run_suite_mode(args, bufs, P, W, torch, stream, peaks, "tf32")
        out["pr1"] = {m: run_pr1(args, P, W, torch, stream, peaks, m) for m in ("3xtf32", "tf32")}
        out["gemm"] = {m: run_gemm_sweep(args, P, W, torch, stream, peaks, m) for m in ("3xtf32", "tf32")}

    # ---- CPU baseline on rank 0, N=1 only
    if rank == 0 and world == 1 and not args.no_cpu:
        gf, reps, secs = cpu_suite_sample(layers, args.cpu_seconds, cpu_cores())
        out["cpu_baseline"] = {"value": round(gf, 2), "unit": "GFLOP/s", "cores": cpu_cores(),
                               "kind": "port",
                               "sample": f"oracle fp32 Fig.9 loop nest (oracle/pdl_oracle.c), "
                                         f"1 image per layer x 20 layers, fused bias+ReLU, "
                                         f"{reps} reps in {secs:.1f} s",
                               "note": "untuned C restatement of the reference nest (OpenMP over "
                                       "images / output-channel tiles); the paper's tuned PolyDL "
                                       "reaches ~2.3 TFLOP/s on 28 Cascade Lake cores "
                                       "(PAPER.md:845-848), so GPU/CPU ratios against this port "
                                       "overstate the gap to a tuned CPU code"}
        try:
            out["cpu_baseline"]["torch_cpu_onednn"] = cpu_torch_onednn(
                layers, min(5.0, args.cpu_seconds), cpu_cores())
        except Exception as e:  # noqa: BLE001 -- a missing CPU backend must not kill the bench
            out["cpu_baseline"]["torch_cpu_onednn"] = {"unavailable": str(e)[:200]}
        ref = reference_interpret_record(total_flops)
        if ref is not None:
            out["cpu_baseline"]["reference_interpret"] = ref
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def compact_x(layer, x):
    """The narrow-channel layer's x as [N][H][W][4] (its real channels + zero padding)."""
    return x[:, 0, :, :, :4].contiguous()


def run_suite_e2e(args, bufs, P, torch, dev, world, dist, total_flops, stream, compact_stem=False):
    """Same metric through the public API with pinned HOST buffers: each step
    copies every layer's x host->device, runs the fused conv, and copies y back.
    Timed over all --steps steps.  compact_stem: layers with C <= 4 (the stem) take
    their host x as [N][H][W][4] instead of nChw16c's 64-byte pixels."""
    srcs = [compact_x(layer, x) if (compact_stem and layer.C <= 4) else x for (layer, x, *_r) in bufs]
    hx = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in srcs]
    hy = [torch.empty(y.shape, dtype=torch.float32, pin_memory=True) for (*_r, y) in bufs]
    for h, x in zip(hx, srcs):
        h.copy_(x)
    del srcs
    h2d = sum(h.numel() * 4 for h in hx)
    d2h = sum(h.numel() * 4 for h in hy)

    def step():
        for (layer, x, w, b, pw, y), xh, yh in zip(bufs, hx, hy):
            # every layer's input is a host array prepared before the step (x_ready):
            # a layer's copies in overlap the previous layer's copies out
            P.conv2d_nchw16c_host(xh, pw, b, stride=layer.stride, pad=layer.pad, relu=True,
                                  mode=args.mode, out=yh, x_ready=True)

    steps = max(1, args.steps)
    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    from paper_2006_02230_b200.shard import max_over_ranks
    ms = max_over_ranks(e0.elapsed_time(e1), dev)
    return {"value": round(total_flops / (ms / steps / 1e3) / 1e9, 1), "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "ms_per_step": round(ms / steps, 3),
            "path": "paper_2006_02230_b200.conv2d_nchw16c_host -> libpdl.so pdl_conv2d_fwd_host "
                    "(pinned host x/y; image chunks pipelined: H2D, fused conv and D2H on three "
                    "streams), every copy inside the timed region"
                    + ("; stem x as [N][H][W][4] (PDL_X_NCHW4C)" if compact_stem else "")}


def run_stem_compact(args, bufs, P, W, torch, stream, peaks, per_layer):
    """The stem with its input in the compact [N][H][W][4] layout (PDL_X_NCHW4C) beside
    the nChw16c call: back-to-back launches of each, alternating, on the suite's stem
    buffers (x + y = 1.0 / 1.6 GB per launch >> L2)."""
    i0 = next((i for i, b in enumerate(bufs) if b[0].C <= 4), None)
    if i0 is None:
        return {"skipped": "no narrow-channel layer"}
    layer, x, w, b, pw, y = bufs[i0]
    n = x.shape[0]
    x4 = compact_x(layer, x)
    mpeak, label = mode_peak(peaks, args.mode)

    def call(xin):
        return lambda: P.conv2d_nchw16c(xin, pw, b, stride=layer.stride, pad=layer.pad, relu=True,
                                        mode=args.mode, out=y, channels=layer.C)
    _, per = time_calls(torch, [call(x), call(x4)], 1, stream, graph=False, per_call=max(5, args.steps))
    y16 = y.clone()
    call(x4)()
    same = bool(torch.equal(y, y16))
    f = layer.flops(n)
    hbm = peaks["hbm_gbs"] * 1e9
    res = {"layer": layer.name(), "bitwise_equal_to_nchw16c": same, "roofline_peak_source": label}
    for key, ms, stored in (("nchw16c", per[0], n * layer.H * layer.W * 64),
                            ("nchw4c", per[1], n * layer.H * layer.W * 16)):
        res[key] = {"ms": round(ms, 4), "gflops": round(f / ms / 1e6, 1),
                    "tensor_frac": round(f / (ms / 1e3) / mpeak, 3),
                    "x_bytes_stored": stored,
                    "hbm_floor_ms": round((stored + n * layer.K * layer.P * layer.Q * 4) / hbm * 1e3, 4)}
    res["speedup"] = round(per[0] / per[1], 3)
    return res


def run_unfused(args, bufs, P, torch, stream):
    res = []
    for layer, x, w, b, pw, y in bufs:
        def fused():
            P.conv2d_nchw16c(x, pw, b, stride=layer.stride, pad=layer.pad, relu=True,
                             mode=args.mode, out=y)

        def unfused():
            P.conv2d_nchw16c(x, pw, None, stride=layer.stride, pad=layer.pad, mode=args.mode, out=y)
            P.bias_relu_(y, b)

        t = {}
        for name, fn in (("fused", fused), ("unfused", unfused)):
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            t[name] = e0.elapsed_time(e1) / 5
        n = x.shape[0]
        res.append({"layer": layer.name(), "fused_ms": round(t["fused"], 4),
                    "unfused_ms": round(t["unfused"], 4),
                    "speedup": round(t["unfused"] / t["fused"], 3),
                    "hbm_bytes_saved": layer.unfused_extra_bytes(n)})
    return res


# ----------------------------------------------------------------------------- other configs
def _packed_for(bufs, P, mode):
    """Per-layer weights prepacked for `mode` (the suite's own when it matches)."""
    out = []
    for layer, x, w, b, pw, y in bufs:
        out.append(pw if pw.mode == mode else P.prepack_weights(w, mode=mode, channels=layer.C))
    return out


def run_n28(args, bufs, P, W, torch, stream, peaks):
    """BASELINE configs[2]/[3]: the 20-layer suite at the paper's minibatch N=28
    (PAPER.md:812-813), fused conv+bias+ReLU and the unfused GPU two-kernel
    baseline (conv, then a separate bias+ReLU pass), in 3xTF32 and TF32.  Each
    pass over the 20 layers is one CUDA-graph replay; the layers' inputs (x[:28] of
    the suite's buffers, 20-layer working set 0.85 GB) do not fit the 126 MB L2."""
    n = 28
    if bufs[0][1].shape[0] < n:
        return {"skipped": f"per-GPU batch {bufs[0][1].shape[0]} < 28"}
    hbm = peaks["hbm_gbs"] * 1e9
    res = {"config": "20 ResNet-50 v1 layers, N=28, fused conv+bias+ReLU vs conv then bias+ReLU pass",
           "steps": args.steps}
    for mode in ("3xtf32", "tf32"):
        mpeak, label = mode_peak(peaks, mode)
        pws = _packed_for(bufs, P, mode)
        fused, unfused = [], []
        for (layer, x, w, b, _pw, y), pw in zip(bufs, pws):
            xs, ys = x[:n], y[:n]
            fused.append(lambda l=layer, xs=xs, pw=pw, b=b, ys=ys: P.conv2d_nchw16c(
                xs, pw, b, stride=l.stride, pad=l.pad, relu=True, mode=mode, out=ys))
            unfused.append(lambda l=layer, xs=xs, pw=pw, ys=ys: P.conv2d_nchw16c(
                xs, pw, None, stride=l.stride, pad=l.pad, mode=mode, out=ys))
            unfused.append(lambda ys=ys, b=b: P.bias_relu_(ys, b))
        tf, per_f = time_calls(torch, fused, args.steps, stream, per_call=3)
        tu, per_u = time_calls(torch, unfused, args.steps, stream, per_call=3)
        flops = sum(b_[0].flops(n) for b_ in bufs)
        rows = []
        for i, (layer, *_r) in enumerate(bufs):
            r = layer_row(W, layer, n, per_f[i], mpeak, hbm)
            r["unfused_ms"] = round(per_u[2 * i] + per_u[2 * i + 1], 4)
            r["speedup_vs_unfused"] = round(r["unfused_ms"] / r["ms"], 3)
            r["hbm_bytes_saved"] = layer.unfused_extra_bytes(n)
            rows.append(r)
        res[mode] = {"fused": {"value": round(flops / (tf / 1e3) / 1e9, 1), "unit": "GFLOP/s",
                               "ms_per_step": round(tf, 4)},
                     "unfused": {"value": round(flops / (tu / 1e3) / 1e9, 1), "unit": "GFLOP/s",
                                 "ms_per_step": round(tu, 4)},
                     "speedup_fused_vs_unfused": round(tu / tf, 3),
                     "hbm_bytes_saved_per_step": sum(b_[0].unfused_extra_bytes(n) for b_ in bufs),
                     "roofline_peak_source": label,
                     "layers_below_0.6": sum(1 for r in rows if r["roofline_frac"] < 0.6),
                     "layers": rows}
    return res


def run_suite_mode(args, bufs, P, W, torch, stream, peaks, mode):
    """The 256-image suite again in another arithmetic mode (TF32: one tensor pass,
    1e-2 bar), same buffers, graph-replayed step."""
    hbm = peaks["hbm_gbs"] * 1e9
    mpeak, label = mode_peak(peaks, mode)
    pws = _packed_for(bufs, P, mode)
    calls = [lambda l=layer, x=x, pw=pw, b=b, y=y: P.conv2d_nchw16c(
        x, pw, b, stride=l.stride, pad=l.pad, relu=True, mode=mode, out=y)
        for (layer, x, w, b, _pw, y), pw in zip(bufs, pws)]
    t, per = time_calls(torch, calls, args.steps, stream, per_call=3)
    n = bufs[0][1].shape[0]
    flops = sum(b_[0].flops(n) for b_ in bufs)
    rows = [layer_row(W, b_[0], n, per[i], mpeak, hbm) for i, b_ in enumerate(bufs)]
    return {"mode": mode, "value": round(flops / (t / 1e3) / 1e9, 1), "unit": "GFLOP/s",
            "ms_per_step": round(t, 4), "global_batch": n, "roofline_peak_source": label,
            "layers_below_0.6": sum(1 for r in rows if r["roofline_frac"] < 0.6), "layers": rows}


def _rotation(set_bytes: int, min_sets: int = 8, budget: int = 320 << 20, cap: int = 256) -> int:
    """Number of rotating input sets so consecutive launches read cold data
    (sets x bytes > the 126 MB L2 where the budget allows)."""
    return max(min_sets, min(cap, -(-budget // max(set_bytes, 1))))


def run_pr1(args, P, W, torch, stream, peaks, mode):
    """BASELINE configs[0]: PR1 (N=1, C=K=64, 56x56, 3x3, s1, p1, no bias).  Back-to-back
    launches (the paper averages repeated runs) over rotated x / y
    buffers (2 x 0.8 MB per launch; the rotation spans > 126 MB L2, so x is cold),
    captured as one CUDA graph; ms = graph time / launches."""
    layer = W.PR1
    mpeak, label = mode_peak(peaks, mode)
    x, w, _ = W.conv_inputs(layer, 1, seed=1234, bias=False)
    xd = torch.from_numpy(x).cuda()
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), mode=mode)
    nrot = _rotation(2 * x.nbytes)
    xs = [xd.clone() for _ in range(nrot)]
    ys = [torch.empty((1, 4, 56, 56, 16), device="cuda") for _ in range(nrot)]
    calls = [lambda i=i: P.conv2d_nchw16c(xs[i], pw, stride=1, pad=1, mode=mode, out=ys[i])
             for i in range(nrot)]
    t, _ = time_calls(torch, calls, max(1, args.steps // 10), stream)
    ms = t / nrot
    f = layer.flops(1)
    rf = W.Roofline(f, layer.bytes(1), mpeak, peaks["hbm_gbs"] * 1e9)
    return {"ms": round(ms, 5), "us": round(ms * 1e3, 2), "gflops": round(f / ms / 1e6, 1),
            "bound": rf.bound, "roofline_frac": round(rf.fraction(ms / 1e3), 4),
            "roofline_peak_source": label,
            "timing": f"{nrot} back-to-back launches per CUDA graph over {nrot} rotated x/y buffers"}


def run_gemm_sweep(args, P, W, torch, stream, peaks, mode, cfg=None):
    """BASELINE configs[1]: the GEMM sweep (row-major fp32, beta = 0).  Per shape:
    back-to-back launches in one CUDA graph over rotated A/B/C sets (>= 8 sets,
    > 126 MB in total where 320 MB allows), ms = graph time / launches."""
    mpeak, label = mode_peak(peaks, mode)
    hbm = peaks["hbm_gbs"] * 1e9
    rows, tot_f, tot_ms = [], 0.0, 0.0
    for (m, n, k) in W.GEMM_SWEEP:
        g = torch.Generator(device="cuda")
        g.manual_seed(m * 31 + n * 7 + k)
        nsets = min(_rotation(W.gemm_bytes(m, n, k)), max(2, (1 << 30) // W.gemm_bytes(m, n, k)))
        a0 = torch.rand((m, k), generator=g, device="cuda") * 2 - 1
        b0 = torch.rand((k, n), generator=g, device="cuda") * 2 - 1
        sets = [(a0.clone(), b0.clone(), torch.empty((m, n), device="cuda")) for _ in range(nsets)]
        nl = max(nsets, 8)
        calls = [lambda s=sets[i % nsets]: P.gemm(s[0], s[1], s[2], mode=mode, cfg=cfg) for i in range(nl)]
        t, _ = time_calls(torch, calls, max(2, args.steps // 10), stream)
        ms = t / nl
        f = W.gemm_flops(m, n, k)
        rf = W.Roofline(f, W.gemm_bytes(m, n, k), mpeak, hbm)
        rows.append({"shape": [m, n, k], "ms": round(ms, 5), "us": round(ms * 1e3, 2),
                     "gflops": round(f / ms / 1e6, 1), "bound": rf.bound,
                     "roofline_frac": round(rf.fraction(ms / 1e3), 4), "sets": nsets, "launches": nl,
                     "l2_cold": nsets * W.gemm_bytes(m, n, k) > (126 << 20)})
        tot_f += f
        tot_ms += ms
        del sets, a0, b0
    return {"value": round(tot_f / tot_ms / 1e6, 1), "unit": "GFLOP/s",
            "aggregate": "total FLOPs of the 10 shapes / summed per-launch times",
            "roofline_peak_source": label, "shapes": rows}


def run_gemm(args, rank, world, local):
    import torch
    import paper_2006_02230_b200 as P
    from paper_2006_02230_b200 import workloads as W
    torch.cuda.set_device(local)
    peaks = load_peaks()
    mpeak, label = mode_peak(peaks, args.mode)
    stream = torch.cuda.current_stream()
    gcfg = {"cluster_m": args.cluster} if args.cluster else None
    sw = run_gemm_sweep(args, P, W, torch, stream, peaks, args.mode, gcfg)
    big = max(sw["shapes"], key=lambda r: r["ms"])
    m, n, k = big["shape"]
    achieved = W.gemm_flops(m, n, k) / (big["ms"] / 1e3) / 1e12
    return {"metric": METRIC, "value": sw["value"], "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sum(r["ms"] for r in sw["shapes"]), 4), "higher_is_better": True,
            "scaling": "replicas only", "vs_baseline": None, "dtype": "f32", "data": "synthetic U[-1,1)",
            "config": {"workload": "gemm_sweep_rowmajor_fp32", "mode": args.mode,
                       "l2": "rotated input sets, > 126 MB per rotation where 320 MB allows"},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 2),
                         "peak": round(mpeak / 1e12, 1), "unit": "TFLOP/s",
                         "frac": round(achieved / (mpeak / 1e12), 4), "peak_source": label,
                         "kernel": f"tile_mma_kernel[gemm {m}x{n}x{k}]", "traffic": None},
            "gemms": sw["shapes"], "gpu_launches": sum(r["launches"] for r in sw["shapes"])}


def run_layout(args, rank, world, local):
    """Data path either side of the conv: NCHW -> nChw16c pack of
    the network input and nChw16c -> NCHW unpack of the largest activation at
    batch 256; HBM-bound, algorithmic bytes = read + write."""
    import torch
    import paper_2006_02230_b200 as P
    torch.cuda.set_device(local)
    peaks = load_peaks()
    n = args.batch
    cases = [("pack_nchw16c stem input", "pack", (n, 3, 224, 224)),
             ("pack_nchw16c 64x56x56", "pack", (n, 64, 56, 56)),
             ("unpack_nchw16c 256x56x56", "unpack", (n, 256, 56, 56)),
             ("unpack_nchw16c 2048x7x7", "unpack", (n, 2048, 7, 7))]
    stream = torch.cuda.current_stream()
    rows, tot_b, tot_ms = [], 0, 0.0
    for name, kind, (N, C, H, Wd) in cases:
        cb = (C + 15) // 16
        nchw = torch.rand((N, C, H, Wd), device="cuda")
        blk = torch.empty((N, cb, H, Wd, 16), device="cuda")
        if kind == "unpack":
            P.to_nchw16c(nchw, out=blk)
        run = (lambda: P.to_nchw16c(nchw, out=blk)) if kind == "pack" else \
            (lambda: P.from_nchw16c(blk, C, out=nchw))
        for _ in range(args.warmup):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        nbytes = 4 * N * C * H * Wd + 4 * N * cb * 16 * H * Wd
        rows.append({"case": name, "ms": round(ms, 4), "gbs": round(nbytes / ms / 1e6, 1),
                     "roofline_frac": round(nbytes / ms / 1e6 / peaks["hbm_gbs"], 3)})
        tot_b += nbytes
        tot_ms += ms
    gbs = tot_b / tot_ms / 1e6
    return {"metric": "NCHW<->nChw16c pack/unpack GB/s", "value": round(gbs, 1), "unit": "GB/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_ms, 4),
            "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic U[0,1)",
            "config": {"workload": "layout_pack_unpack", "batch": n,
                       "l2": "every tensor >> 126 MB L2 except 2048x7x7 (102 MB)"},
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": round(gbs / peaks["hbm_gbs"], 4),
                         "kernel": "pack_nchw16c_kernel / unpack_nchw16c_kernel", "traffic": None},
            "cases": rows, "gpu_launches": len(rows) * (args.steps + args.warmup)}


def run_suite_pr1(args, rank, world, local):
    """PR1 alone (configs[0]) as a bench line."""
    import torch
    import paper_2006_02230_b200 as P
    from paper_2006_02230_b200 import workloads as W
    torch.cuda.set_device(local)
    peaks = load_peaks()
    r = run_pr1(args, P, W, torch, torch.cuda.current_stream(), peaks, args.mode)
    return {"metric": METRIC, "value": r["gflops"], "unit": "GFLOP/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms"],
            "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic U[-1,1) seed 1234",
            "config": {"workload": "PR1 conv 3x3 N=1 C=K=64 56x56", "mode": args.mode,
                       "l2": r["timing"]},
            "roofline": {"bound": r["bound"], "frac": r["roofline_frac"],
                         "peak_source": r["roofline_peak_source"]},
            "gpu_launches": None}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's CPU implementation of the path = the oracle port of the
    Fig. 9 loop nest (the reference itself is a Python interpreter that cannot
    travel to the box).  Rank 0 only."""
    if rank != 0:
        return None
    from paper_2006_02230_b200 import workloads as W
    cores = cpu_cores()
    layers = W.LAYERS
    flops = sum(l.flops(1) for l in layers)
    prepared = cpu_prepare(layers)
    for _ in range(args.warmup):
        cpu_step(prepared, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_step(prepared, cores)
    secs = time.perf_counter() - t0
    value = flops * args.steps / secs / 1e9
    sample = ("oracle fp32 Fig.9 loop nest, 1 image per layer x 20 ResNet-50 layers, fused "
              "bias+ReLU, per step")
    return {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(secs / args.steps * 1e3, 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded U[-1,1))",
            "config": {"workload": "resnet50_v1_20_distinct_layers_fused_conv_bias_relu",
                       "global_batch": args.batch, "mode": "fp32 (CPU)",
                       "sample_per_step": "1 image per layer"},
            "cpu_baseline": {"value": round(value, 2), "unit": "GFLOP/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    rank, world, local = dist_info()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    elif args.workload == "suite":
        out = run_suite(args, rank, world, local)
    elif args.workload == "gemm":
        out = run_gemm(args, rank, world, local) if rank == 0 else None
    elif args.workload == "layout":
        out = run_layout(args, rank, world, local) if rank == 0 else None
    else:
        out = run_suite_pr1(args, rank, world, local) if rank == 0 else None
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
