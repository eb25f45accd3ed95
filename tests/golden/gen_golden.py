"""Generate golden vectors by running the UNMODIFIED reference interpreter.

Container-only (needs /root/reference).  Imports `looprank` read-only and runs
`looprank.simcache.interpret` (reference simcache.py:89-204) on the Fig. 9
blocked-conv nest, the Fig. 1 GEMM nest
and the conv -> bias+ReLU program (SURVEY Appendix C.2 shape), on seeded
U[-1,1) fp32-valued inputs with zeroed outputs.  Results are float64 arrays
saved as .npz fixtures next to this script; the `.pdl` source text is stored
in each fixture so the host-side parser is exercised on the same programs.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/gen_golden.py [--pr1]

`--pr1` additionally runs the full PR1 layer (N=1, C=K=64, 56x56, 3x3, s1, p1;
115.6 M MAC, ~20-40 min) and stores the SHA-256 of the float64 output bytes
plus summary statistics (the full output is not committed).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from looprank import loopdsl, simcache  # noqa: E402


def conv_pdl(stride: int, relu: bool) -> str:
    s = stride
    txt = f"""param N, KT, CT, P, Q, R, S;
array output[N][KT][P][Q][16];
array filter[KT][CT][R][S][16][16];
array input[N][CT][{s}*P - {s} + R][{s}*Q - {s} + S][16];
conv: parallel for (img = 0; img < N; img++) {{
  for (ofm_tile = 0; ofm_tile < KT; ofm_tile++) {{
    for (ifm_tile = 0; ifm_tile < CT; ifm_tile++) {{
      for (oj = 0; oj < P; oj++) {{
        ij = oj * {s};
        for (kj = 0; kj < R; kj++) {{
          for (ki = 0; ki < S; ki++) {{
            #pragma microkernel gemm(output, filter, input)
            {{
              for (oi = 0; oi < Q; oi++) {{
                ii = oi * {s};
                for (ofm = 0; ofm < 16; ofm++) {{
                  for (ifm = 0; ifm < 16; ifm++) {{
                    Sc: output[img][ofm_tile][oj][oi][ofm] += filter[ofm_tile][ifm_tile][kj][ki][ifm][ofm] * input[img][ifm_tile][ij + kj][ii + ki][ifm];
                  }}
                }}
              }}
            }}
          }}
        }}
      }}
    }}
  }}
}}
"""
    if relu:
        txt += """array bias[KT][16];
relu: parallel for (img2 = 0; img2 < N; img2++) {
  for (t2 = 0; t2 < KT; t2++) {
    for (p2 = 0; p2 < P; p2++) {
      for (q2 = 0; q2 < Q; q2++) {
        for (v2 = 0; v2 < 16; v2++) {
          T: output[img2][t2][p2][q2][v2] = max(output[img2][t2][p2][q2][v2] + bias[t2][v2], 0.0);
        }
      }
    }
  }
}
"""
    return txt


GEMM_PDL = """param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
gemm: parallel for (i = 0; i < M; i++) {
  for (j = 0; j < N; j++) {
    for (k = 0; k < K; k++) {
      S: C[i][j] += A[i][k] * B[k][j];
    }
  }
}
"""


def u(rng, shape, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def make_conv_case(seed, n, c, k, h, w, r, s_, stride, pad, relu, real_c=None):
    """Unpadded nChw16c input, KCRS16c16k weights, bias [K]; fp32 values."""
    ct, kt = c // 16, k // 16
    x = u(np.random.default_rng(seed), (n, ct, h, w, 16))
    if real_c is not None:  # stem: real channels then zero padding
        mask = np.zeros((ct, 16), np.float32)
        mask.reshape(-1)[:real_c] = 1.0
        x *= mask[None, :, None, None, :]
    wt = u(np.random.default_rng(seed + 1), (kt, ct, r, s_, 16, 16))
    b = u(np.random.default_rng(seed + 2), (kt, 16), -0.5, 0.5)
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - s_) // stride + 1
    return x, wt, b, p, q


def run_conv(name, seed, n, c, k, h, w, r, s_, stride, pad, relu=False, real_c=None):
    x, wt, b, p, q = make_conv_case(seed, n, c, k, h, w, r, s_, stride, pad, relu, real_c)
    kt, ct = k // 16, c // 16
    hp = stride * p - stride + r
    wp = stride * q - stride + s_
    xp = np.zeros((n, ct, hp, wp, 16), np.float32)
    hh = min(h, hp - pad)
    ww = min(w, wp - pad)
    xp[:, :, pad:pad + hh, pad:pad + ww, :] = x[:, :, :hh, :ww, :]
    text = conv_pdl(stride, relu)
    binding = dict(N=n, KT=kt, CT=ct, P=p, Q=q, R=r, S=s_)
    inputs = {"output": np.zeros((n, kt, p, q, 16)), "filter": wt, "input": xp}
    t0 = time.time()
    if relu:
        prog = loopdsl.parse_program(text)
        inputs["bias"] = b
        arrays, _ = simcache.interpret(prog.nests[0], binding, inputs=inputs, collect_trace=False)
        arrays, _ = simcache.interpret(prog.nests[1], binding, inputs=arrays, collect_trace=False)
    else:
        nest = loopdsl.parse(text)
        arrays, _ = simcache.interpret(nest, binding, inputs=inputs, collect_trace=False)
    dt = time.time() - t0
    y = arrays["output"].reshape(n, kt, p, q, 16)
    out = dict(kind="conv", text=text, x=x, w=wt, y=y, N=n, C=c, K=k, H=h, W=w, R=r, S=s_,
               stride=stride, pad=pad, relu=int(relu), seed=seed)
    if relu:
        out["bias"] = b.reshape(-1)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {dt:.1f}s  |y|max={np.abs(y).max():.4f}", flush=True)


def run_gemm(name, seed, m, n, k):
    a = u(np.random.default_rng(seed), (m, k))
    b = u(np.random.default_rng(seed + 1), (k, n))
    nest = loopdsl.parse(GEMM_PDL)
    t0 = time.time()
    arrays, _ = simcache.interpret(nest, dict(M=m, N=n, K=k),
                                   inputs={"C": np.zeros((m, n)), "A": a, "B": b},
                                   collect_trace=False)
    dt = time.time() - t0
    c = arrays["C"].reshape(m, n)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), kind="gemm", text=GEMM_PDL,
                        A=a, B=b, C=c, M=m, N=n, K=k, seed=seed)
    print(f"{name}: {dt:.1f}s", flush=True)


def run_pr1(seed=1234):
    n, c, k, h, w, r, s_, stride, pad = 1, 64, 64, 56, 56, 3, 3, 1, 1
    x, wt, b, p, q = make_conv_case(seed, n, c, k, h, w, r, s_, stride, pad, False)
    xp = np.zeros((n, c // 16, h + 2, w + 2, 16), np.float32)
    xp[:, :, 1:-1, 1:-1, :] = x
    nest = loopdsl.parse(conv_pdl(1, False))
    binding = dict(N=n, KT=k // 16, CT=c // 16, P=p, Q=q, R=r, S=s_)
    t0 = time.time()
    arrays, _ = simcache.interpret(nest, binding,
                                   inputs={"output": np.zeros((n, k // 16, p, q, 16)),
                                           "filter": wt, "input": xp},
                                   collect_trace=False)
    dt = time.time() - t0
    y = np.ascontiguousarray(arrays["output"], dtype=np.float64)
    rec = dict(config="PR1", seed=seed, N=n, C=c, K=k, H=h, W=w, R=r, S=s_, stride=stride,
               pad=pad, inputs="x=U[-1,1) rng(seed) shape (1,4,56,56,16) fp32; "
                               "w=U[-1,1) rng(seed+1) shape (4,4,3,3,16,16) fp32",
               sha256_f64=hashlib.sha256(y.tobytes()).hexdigest(),
               sum=float(y.sum()), abs_max=float(np.abs(y).max()),
               first8=[float(v) for v in y[:8]], interpret_seconds=round(dt, 1),
               numpy=np.__version__)
    with open(os.path.join(HERE, "pr1_interpret.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(f"PR1: {dt:.1f}s sha={rec['sha256_f64'][:16]}", flush=True)


CASES = [
    ("conv_3x3_s1", dict(seed=11, n=2, c=32, k=32, h=6, w=6, r=3, s_=3, stride=1, pad=1)),
    ("conv_1x1_s1", dict(seed=12, n=2, c=32, k=48, h=5, w=5, r=1, s_=1, stride=1, pad=0)),
    ("conv_1x1_s2", dict(seed=13, n=2, c=32, k=32, h=8, w=8, r=1, s_=1, stride=2, pad=0)),
    ("conv_3x3_s2", dict(seed=14, n=1, c=16, k=16, h=7, w=7, r=3, s_=3, stride=2, pad=1)),
    ("conv_7x7_s2_stem", dict(seed=15, n=1, c=16, k=32, h=12, w=12, r=7, s_=7, stride=2,
                              pad=3, real_c=3)),
    ("conv_3x3_s1_relu", dict(seed=16, n=1, c=32, k=32, h=5, w=5, r=3, s_=3, stride=1, pad=1,
                              relu=True)),
    ("conv_1x1_s1_relu", dict(seed=17, n=2, c=16, k=32, h=7, w=7, r=1, s_=1, stride=1, pad=0,
                              relu=True)),
]
GEMMS = [("gemm_16", dict(seed=21, m=16, n=16, k=16)),
         ("gemm_ragged", dict(seed=22, m=37, n=45, k=29)),
         ("gemm_tall", dict(seed=23, m=130, n=8, k=24))]

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--pr1", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    if args.pr1:
        run_pr1()
        sys.exit(0)
    for name, kw in CASES:
        if args.only and args.only != name:
            continue
        run_conv(name, **kw)
    for name, kw in GEMMS:
        if args.only and args.only != name:
            continue
        run_gemm(name, **kw)
