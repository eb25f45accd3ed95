"""Golden vectors for the Alg. 3 fusion pass, made by the UNMODIFIED reference.

Container-only (needs /root/reference).  For each case the two-operator program
is fused by paper_2006_02230_b200.fusion.fuse, the fused nest is printed as
`.pdl` text, and that text is parsed and run by the reference's own
`looprank.loopdsl.parse` + `looprank.simcache.interpret` (simcache.py:89-204);
the unfused program is run the same way, nest by nest.  Stored per case: both
texts, the binding, the inputs and both reference outputs (float64), so the CPU
tests check the fused nest against the reference's execution of it, and the
semantic-preservation invariant (fused == unfused, bitwise) on the reference's
own arithmetic.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \\
        python tests/golden/gen_fusion.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from looprank import loopdsl, simcache  # noqa: E402

from paper_2006_02230_b200 import fusion as F  # noqa: E402
from paper_2006_02230_b200 import loopnest as L  # noqa: E402

GEMM_EW = """param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
array s[N];
array t[N];
gemm: for (i = 0; i < M; i++) {{
  for (j = 0; j < N; j++) {{
    for (k = 0; k < K; k++) {{
      S: C[i][j] += A[i][k] * B[k][j];
    }}
  }}
}}
ew: for (i2 = 0; i2 < M; i2++) {{
  for (j2 = 0; j2 < N; j2++) {{
    E: C[i2][j2] = {expr};
  }}
}}
"""

EW_GEMM = """param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
ew: for (i2 = 0; i2 < M; i2++) {
  for (j2 = 0; j2 < N; j2++) {
    E: C[i2][j2] = max(C[i2][j2], 0.0);
  }
}
gemm: for (i = 0; i < M; i++) {
  for (k = 0; k < K; k++) {
    for (j = 0; j < N; j++) {
      S: C[i][j] += A[i][k] * B[k][j];
    }
  }
}
"""

CONV_EW = """param N, KT, CT, P, Q, R, S;
array output[N][KT][P][Q][16];
array filter[KT][CT][R][S][16][16];
array input[N][CT][P + R - 1][Q + S - 1][16];
array bias[KT][16];
array scale[KT][16];
conv: parallel for (img = 0; img < N; img++) {{
  for (ofm_tile = 0; ofm_tile < KT; ofm_tile++) {{
    for (ifm_tile = 0; ifm_tile < CT; ifm_tile++) {{
      for (oj = 0; oj < P; oj++) {{
        for (kj = 0; kj < R; kj++) {{
          for (ki = 0; ki < S; ki++) {{
            for (oi = 0; oi < Q; oi++) {{
              for (ofm = 0; ofm < 16; ofm++) {{
                for (ifm = 0; ifm < 16; ifm++) {{
                  Sc: output[img][ofm_tile][oj][oi][ofm] += filter[ofm_tile][ifm_tile][kj][ki][ifm][ofm] * input[img][ifm_tile][oj + kj][oi + ki][ifm];
                }}
              }}
            }}
          }}
        }}
      }}
    }}
  }}
}}
act: parallel for (img2 = 0; img2 < N; img2++) {{
  for (t2 = 0; t2 < KT; t2++) {{
    for (p2 = 0; p2 < P; p2++) {{
      for (q2 = 0; q2 < Q; q2++) {{
        for (v2 = 0; v2 < 16; v2++) {{
          T: output[img2][t2][p2][q2][v2] = {expr};
        }}
      }}
    }}
  }}
}}
"""

Y2 = "C[i2][j2]"
Y5 = "output[img2][t2][p2][q2][v2]"


def cases():
    yield ("gemm_relu_k4", GEMM_EW.format(expr=f"max({Y2}, 0.0)"), dict(M=3, N=5, K=4), False)
    yield ("gemm_relu6_k1", GEMM_EW.format(expr=f"min(max({Y2}, 0.0), 6.0)"), dict(M=4, N=3, K=1), False)
    yield ("gemm_bnorm_relu", GEMM_EW.format(expr=f"max({Y2} * s[j2] + t[j2], 0.0)"),
           dict(M=3, N=4, K=6), False)
    yield ("relu_then_gemm", EW_GEMM, dict(M=3, N=4, K=5), True)
    yield ("conv_relu6", CONV_EW.format(expr=f"min(max({Y5} + bias[t2][v2], 0.0), 6.0)"),
           dict(N=1, KT=2, CT=1, P=3, Q=3, R=3, S=3), False)
    yield ("conv_bnorm_relu", CONV_EW.format(expr=f"max({Y5} * scale[t2][v2] + bias[t2][v2], 0.0)"),
           dict(N=2, KT=1, CT=2, P=2, Q=3, R=1, S=1), False)


def ref_run(text: str, binding: dict, inputs: dict) -> dict:
    arrays = {k: np.array(v, np.float64) for k, v in inputs.items()}
    prog = loopdsl.parse_program(text)
    for nest in prog.nests:
        arrays, _ = simcache.interpret(nest, binding, inputs=arrays, collect_trace=False)
    return arrays


def main() -> None:
    out = {}
    for name, text, binding, ew_first in cases():
        prog = L.parse_program(text)
        a, b = prog.nests
        pair = F.OperatorPair(b, a, ew_first=True) if ew_first else F.OperatorPair(a, b)
        fused_text = L.pretty(F.fuse(pair, binding))
        shapes = {}
        for n in prog.nests:
            shapes.update(n.shapes(binding))
        rng = np.random.default_rng(len(out) + 11)
        # outputs start at random values too: the element-wise-first case reads them
        inputs = {k: rng.uniform(-4, 4, int(np.prod(v))).astype(np.float32).astype(np.float64)
                  for k, v in sorted(shapes.items())}
        unfused = ref_run(text, binding, inputs)
        fused = ref_run(fused_text, binding, inputs)
        out[name] = {"text": text, "fused_text": fused_text, "binding": binding, "ew_first": ew_first,
                     "inputs": {k: v.tolist() for k, v in inputs.items()},
                     "unfused": {k: np.asarray(v).ravel().tolist() for k, v in unfused.items()},
                     "fused": {k: np.asarray(v).ravel().tolist() for k, v in fused.items()}}
        same = all(np.array_equal(unfused[k], fused[k]) for k in unfused)
        print(f"{name}: reference fused == unfused: {same}")
    with open(os.path.join(HERE, "fusion_ref.json"), "w") as f:
        json.dump(out, f, sort_keys=True)


if __name__ == "__main__":
    main()
