"""Golden access traces from the UNMODIFIED reference interpreter (container only).

Runs `looprank.simcache.interpret(..., collect_trace=True)` (reference
simcache.py:89-204) on small instances of the Fig. 9 conv nest (with its
`#pragma microkernel gemm` band), the conv -> bias+ReLU program's ReLU nest, and
the GEMM nest, and stores each trace's length, footprint and the SHA-256 of its
`Trace.dump()` text in trace_ref.json.  tests/test_trace.py requires the host
trace walk (paper_2006_02230_b200.trace) to reproduce them byte for byte.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_trace.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from looprank import loopdsl, simcache  # noqa: E402

from gen_golden import GEMM_PDL, conv_pdl  # noqa: E402

CASES = [
    ("conv_s1", lambda: conv_pdl(1, False), 0, dict(N=1, KT=1, CT=1, P=2, Q=3, R=3, S=3)),
    ("conv_s2", lambda: conv_pdl(2, False), 0, dict(N=2, KT=1, CT=2, P=2, Q=2, R=1, S=1)),
    ("relu_nest", lambda: conv_pdl(1, True), 1, dict(N=1, KT=2, CT=1, P=2, Q=2, R=1, S=1)),
    ("gemm", lambda: GEMM_PDL, 0, dict(M=5, N=4, K=3)),
]


def main():
    out = {}
    for name, text, which, binding in CASES:
        prog = loopdsl.parse_program(text())
        nest = prog.nests[which]
        _, tr = simcache.interpret(nest, binding, seed=0, collect_trace=True)
        d = tr.dump()
        out[name] = {"text": text(), "nest": which, "binding": binding, "len": len(tr),
                     "footprint": tr.footprint(), "sha256": hashlib.sha256(d.encode()).hexdigest(),
                     "head": d.splitlines()[:4]}
        print(name, len(tr), tr.footprint())
    with open(os.path.join(HERE, "trace_ref.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
