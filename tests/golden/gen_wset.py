"""Working-set golden vectors from the UNMODIFIED reference (Alg. 1).

Container-only (needs /root/reference).  Runs `looprank.wset.working_sets`
(reference wset.py:166-207) on small loop nests at desk-size bindings and
stores every entry (dependence id, kind, array, variant, elements) plus the
reference's run time in tests/golden/wset_ref.json.  tests/test_rank.py pins
`paper_2006_02230_b200.wset.working_sets` to these, entry for entry.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/gen_wset.py
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)
sys.dont_write_bytecode = True

from gen_golden import conv_pdl  # noqa: E402

GEMM = """param M, N, K;
array C[M][N]; array A[M][K]; array B[K][N];
gemm: {par}for (i = 0; i < M; i++) {{
  for (j = 0; j < N; j++) {{
    for (k = 0; k < K; k++) {{
      S: C[i][j] += A[i][k] * B[k][j];
}} }} }}
"""

TILED = """param M, N, K;
array C[M][N]; array A[M][K]; array B[K][N];
g: parallel for (it = 0; it < M; it += 2) {
  for (kt = 0; kt < K; kt += 2) {
    for (j = 0; j < N; j++) {
      for (ii = 0; ii < 2; ii++) {
        for (kk = 0; kk < 2; kk++) {
          S: C[it + ii][j] += B[kt + kk][j] * A[it + ii][kt + kk];
} } } } }
"""

TWO_STMT = """param N;
array x[N]; array y[N]; array z[N];
t: for (i = 0; i < N; i++) {
  S1: y[i] = x[i] * 2.0;
  S2: z[i] = y[i] + x[i];
}
"""

STENCIL = """param N, T;
array a[N];
st: for (t = 0; t < T; t++) {
  for (i = 1; i < N - 1; i++) {
    S: a[i] = a[i - 1] + a[i + 1];
  }
}
"""

# Sibling parallel loops under one sequential loop, the iterator name `i` reused: the
# S1 -> S2 dependence spans the common parallel iterator i, and WS_par is taken over
# the SOURCE statement's outermost parallel iterator p (reference depend.py:158-159).
SIBLING_PAR = """param N;
array a[N][N]; array b[N];
t: for (s = 0; s < 2; s++) {
  parallel for (p = 0; p < 2; p++) {
    parallel for (i = 0; i < N; i++) {
      S1: a[p][i] = b[i] * 2.0;
    }
  }
  parallel for (i = 0; i < N; i++) {
    S2: b[i] = a[0][N - 1 - i] + 1.0;
  }
}
"""

CASES = [
    ("gemm_seq_333", GEMM.format(par=""), {"M": 3, "N": 3, "K": 3}),
    ("gemm_seq_444", GEMM.format(par=""), {"M": 4, "N": 4, "K": 4}),
    ("gemm_seq_865", GEMM.format(par=""), {"M": 8, "N": 6, "K": 5}),
    ("gemm_seq_5711", GEMM.format(par=""), {"M": 5, "N": 7, "K": 11}),
    ("gemm_par_444", GEMM.format(par="parallel "), {"M": 4, "N": 4, "K": 4}),
    ("gemm_tiled_444", TILED, {"M": 4, "N": 4, "K": 4}),
    ("two_stmt_6", TWO_STMT, {"N": 6}),
    ("stencil_6x3", STENCIL, {"N": 6, "T": 3}),
    ("conv_3x3_tiny", conv_pdl(1, False).replace("16", "2"),
     {"N": 1, "KT": 1, "CT": 1, "P": 2, "Q": 2, "R": 3, "S": 3}),
    ("conv_1x1_s2_tiny", conv_pdl(2, False).replace("16", "2"),
     {"N": 1, "KT": 1, "CT": 1, "P": 2, "Q": 2, "R": 1, "S": 1}),
    ("sibling_par_4", SIBLING_PAR, {"N": 4}),
]


def _run(text, binding, q):
    from looprank import depend, loopdsl, wset
    t = time.time()
    nest = loopdsl.parse(text)
    if nest.has_kernel_call():
        nest = loopdsl.substitute_microkernel(nest)
    rep = wset.working_sets(nest, binding)
    elapsed = round(time.time() - t, 3)
    info = loopdsl.extract_polyhedral(nest)
    deps = [depend.classify_parallel_span(d, info, binding) for d in depend.compute_dependences(info)]
    deps = [d for d in deps if d.relation.domain().lexmin(binding) is not None]  # non-empty under b
    domains = {}
    for st in info.statements:
        lo, hi = st.space.lexmin(binding), st.space.lexmax(binding)
        domains[st.label] = {"cardinality": st.space.cardinality(binding),
                             "lexmin": None if lo is None else [int(v) for v in lo],
                             "lexmax": None if hi is None else [int(v) for v in hi],
                             "vars": list(st.space.vars)}
    q.put({"elapsed_s": elapsed,
           "entries": [[e.dep_id, e.kind, e.array, e.variant, e.elements] for e in rep.entries],
           "deps": [[d.dep_id, d.kind, d.array, d.spans_parallel, d.parallel_iterator] for d in deps],
           "domains": domains})


def main():
    """`--only NAME ...` regenerates just those cases, keeping the others' records."""
    only = sys.argv[sys.argv.index("--only") + 1:] if "--only" in sys.argv else None
    out = {"generator": "looprank.wset.working_sets (reference, unmodified)", "cases": []}
    if only:
        with open(os.path.join(HERE, "wset_ref.json")) as fh:
            out = json.load(fh)
        out["cases"] = [c for c in out["cases"] if c["name"] not in only]
    for name, text, binding in CASES:
        if only and name not in only:
            continue
        q = mp.Queue()
        p = mp.Process(target=_run, args=(text, binding, q))
        p.start()
        p.join(1800)
        if p.is_alive():
            p.kill()
            print(f"{name}: reference timed out, skipped", flush=True)
            continue
        if p.exitcode != 0:
            print(f"{name}: reference failed (exit {p.exitcode}), skipped", flush=True)
            continue
        res = q.get()
        print(f"{name}: {len(res['entries'])} entries in {res['elapsed_s']} s", flush=True)
        out["cases"].append({"name": name, "text": text, "binding": binding, **res})
    with open(os.path.join(HERE, "wset_ref.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
