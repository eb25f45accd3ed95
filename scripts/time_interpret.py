"""Time the UNMODIFIED reference interpreter (looprank.simcache.interpret,
/root/reference/pkg/src/looprank/simcache.py:89-204) on reduced instances of
every BASELINE config class, in this container (it cannot travel to the GPU
box: /root/reference is absent there).  Writes profiles/interpret_ref_r2.json,
which bench.py reports beside its own CPU baselines (SURVEY 8(d) CPU baseline
item 1: "report us/MAC, extrapolated, labelled").

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python scripts/time_interpret.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from looprank import loopdsl, simcache  # noqa: E402

from gen_golden import GEMM_PDL, conv_pdl  # noqa: E402


def time_conv(stride, R, CT, KT, P, Q, relu):
    S = R
    prog = loopdsl.parse_program(conv_pdl(stride, relu))
    b = dict(N=1, KT=KT, CT=CT, P=P, Q=Q, R=R, S=S)
    H, W = stride * P - stride + R, stride * Q - stride + S
    rng = np.random.default_rng(0)
    inputs = {"input": rng.uniform(-1, 1, (1, CT, H, W, 16)),
              "filter": rng.uniform(-1, 1, (KT, CT, R, S, 16, 16)),
              "output": np.zeros((1, KT, P, Q, 16))}
    if relu:
        inputs["bias"] = rng.uniform(-0.5, 0.5, (KT, 16))
    macs = KT * CT * P * Q * R * S * 256
    t0 = time.perf_counter()
    for nest in prog.nests:
        out, _ = simcache.interpret(nest, b, inputs=inputs, collect_trace=False)
        inputs = dict(inputs, **out)
    dt = time.perf_counter() - t0
    return macs, dt


def time_gemm(n):
    nest = loopdsl.parse(GEMM_PDL)
    rng = np.random.default_rng(0)
    inputs = {"A": rng.uniform(-1, 1, (n, n)), "B": rng.uniform(-1, 1, (n, n)), "C": np.zeros((n, n))}
    t0 = time.perf_counter()
    simcache.interpret(nest, {"M": n, "N": n, "K": n}, inputs=inputs, collect_trace=False)
    return n ** 3, time.perf_counter() - t0


def main():
    rows = []
    for name, args in (("conv 3x3 s1 (PR1 class)", (1, 3, 1, 1, 4, 4, False)),
                       ("conv 1x1 s1", (1, 1, 2, 1, 8, 8, False)),
                       ("conv 1x1 s2", (2, 1, 2, 1, 6, 6, False)),
                       ("conv 3x3 s1 + bias/ReLU nest", (1, 3, 1, 1, 4, 4, True)),
                       ("conv 7x7 s2 (stem class)", (2, 7, 1, 1, 2, 2, False))):
        macs, dt = time_conv(*args)
        rows.append({"case": name, "macs": macs, "seconds": round(dt, 3),
                     "us_per_mac": round(dt / macs * 1e6, 3)})
        print(rows[-1], flush=True)
    try:
        macs, dt = time_gemm(24)
        rows.append({"case": "gemm 24^3", "macs": macs, "seconds": round(dt, 3),
                     "us_per_mac": round(dt / macs * 1e6, 3)})
        print(rows[-1], flush=True)
    except Exception as e:  # gemm_pdl signature differences
        print("gemm skipped:", e)
    conv = [r["us_per_mac"] for r in rows if r["case"].startswith("conv")]
    out = {"what": "unmodified looprank.simcache.interpret, collect_trace=False, single-threaded "
                   "Python float64, reduced instances (N=1, one 16-channel block)",
           "where": "build container (no GPU; %d host cores, 1 used)" % os.cpu_count(),
           "cases": rows,
           "conv_us_per_mac_median": float(np.median(conv)),
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    path = os.path.join(ROOT, "profiles", "interpret_ref_r2.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
