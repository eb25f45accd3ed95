"""Pipeline driver (the reference's `cli` module), B200 form:
parse -> substitute microkernel -> recognise the conv / GEMM band -> generate
tile variants -> working sets + Alg. 2 -> rank (Eq. 1 cost, fitted pipeline
model, DNN judge) -> emit launch configs for the top k.

    python -m paper_2006_02230_b200 analyze conv.pdl --bind N=1,KT=1,...
    python -m paper_2006_02230_b200 rank    conv.pdl --bind ... --method both --top-k 3 --out DIR
    python -m paper_2006_02230_b200 emit    conv.pdl --bind ... --variant bn64_bk32_c1_3xtf32
    python -m paper_2006_02230_b200 fuse    prog.pdl --bind ...
    python -m paper_2006_02230_b200 train   pairs.csv --out model.npz
    python -m paper_2006_02230_b200 run     prog.pdl --bind ... [--mode tf32]      (GPU)

Exit codes as the SPEC: 0 success, 1 usage, 2 parse error, 3 analysis error.
Reports are versioned JSON, byte-identical for identical inputs; a human
summary goes to stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

from . import loopnest as L

REPORT_VERSION = 1


class _Usage(Exception):
    pass


def _bindings(text: str) -> dict:
    out = {}
    for part in filter(None, (text or "").split(",")):
        if "=" not in part:
            raise _Usage(f"bad --bind item {part!r} (want NAME=INT)")
        k, v = part.split("=", 1)
        try:
            out[k.strip()] = int(v)
        except ValueError as exc:
            raise _Usage(f"bad --bind value {part!r}") from exc
    return out


def _load(path: str):
    with open(path) as fh:
        text = fh.read()
    return L.parse_program(text).nests


def _dump(obj, path: str | None):
    blob = json.dumps(obj, indent=1, sort_keys=True) + "\n"
    if path:
        with open(path, "w") as fh:
            fh.write(blob)
    return blob


def _workload(nests, binding):
    """The conv / GEMM band of the program as a rankable shape."""
    from .executor import ConvPlan, GemmPlan, plan_program
    from .workloads import ConvShape, GemmShape
    plans = plan_program(nests, binding)
    heavy = [p for p in plans if isinstance(p, (ConvPlan, GemmPlan))]
    if not heavy:
        raise ValueError("no conv or GEMM band found")
    p = heavy[0]
    if isinstance(p, GemmPlan):
        return GemmShape(p.M, p.N, p.K), 1, plans
    # the .pdl input is pre-padded: the kernel runs it with pad 0
    return ConvShape(p.CT * 16, p.KT * 16, p.Hp, p.Wp, p.R, p.S, p.stride, 0), p.N, plans


def cmd_analyze(a) -> int:
    from . import depend, wset
    out = {"version": REPORT_VERSION, "file": os.path.basename(a.file), "binding": a.binding,
           "nests": []}
    for nest in _load(a.file):
        info = depend.extract_polyhedral(nest)
        deps = [depend.classify_parallel_span(d, info, a.binding)
                for d in depend.compute_dependences(info, a.binding)]
        rep = wset.working_sets(nest, a.binding, limit=a.limit)
        out["nests"].append({
            "nest": nest.name,
            "statements": {s.label: {"iterators": list(s.loop_iters),
                                     "parallel": list(s.parallel_iters),
                                     "instances": depend.domain_size(info, s.label, a.binding)}
                           for s in info.statements},
            "dependences": [{"id": d.dep_id, "kind": d.kind, "array": d.array,
                             "spans_parallel": d.spans_parallel} for d in deps],
            "working_sets": rep.to_dict()})
        print(f"{nest.name}: {len(deps)} dependences, {len(rep.entries)} working-set entries, "
              f"{rep.summary()['total_bytes']} bytes total")
    _dump(out, a.out and os.path.join(a.out, "analysis.json"))
    return 0


def cmd_rank(a) -> int:
    from . import rank, variants
    from .machine import default_machine, load_machine
    shape, n, _ = _workload(_load(a.file), a.binding)
    m = load_machine(a.machine) if a.machine else default_machine()
    vs = variants.generate_variants(shape, variants.VariantConfig(modes=(a.mode,)), n_images=n)
    if not vs:
        raise ValueError("no legal variant")
    k = a.top_k
    if k > len(vs):
        print(f"warning: top-k {k} > {len(vs)} variants; emitting all", file=sys.stderr)
        k = len(vs)
    stats = {v.vid: rank.stats_for_variant(shape, v, n, m) for v in vs}
    orders = {}
    if a.method in ("cost", "both"):
        orders["cost"] = rank.rank_by_cost(list(stats.values()), m).to_dict()
    if a.method in ("model", "both"):
        orders["model"] = rank.rank_by_model(shape, vs, n).to_dict()
    if a.method in ("dnn", "both"):
        pm = rank.PipelineModel.load()
        judge = rank.RankerModel.load(a.model) if a.model else None
        best = rank.choose_variant(shape, n, a.mode, method="dnn", judge=judge)
        terms = [pm.term_stats(shape, v, n) for v in vs]
        t = rank.tournament_rank(judge or rank.RankerModel.load(rank._RANKER_FILE), terms,
                                 both_directions=True)
        orders["dnn"] = dict(t.to_dict(), pick=best.vid)
    primary = orders.get("dnn") or orders.get("model") or orders["cost"]
    top = primary.get("pick") and [primary["pick"]] + [v for v in primary["order"] if v != primary["pick"]]
    top = (top or primary["order"])[:k]
    by_id = {v.vid: v for v in vs}
    report = {"version": REPORT_VERSION, "file": os.path.basename(a.file), "binding": a.binding,
              "workload": shape.name(), "images": n, "machine": m.name, "mode": a.mode,
              "variants": {v.vid: {"bn": v.bn, "bk": v.bk, "cluster": v.cluster,
                                   "stats": stats[v.vid].vector().tolist()} for v in vs},
              "rankings": orders,
              "emitted": [{"variant": vid, "launch": variants.emit_launch(by_id[vid])} for vid in top]}
    _dump(report, a.out and os.path.join(a.out, "rank.json"))
    print(f"{shape.name()} x{n}: {len(vs)} variants; top {k}: {', '.join(top)}")
    return 0


def cmd_emit(a) -> int:
    from . import variants
    shape, n, _ = _workload(_load(a.file), a.binding)
    vs = {v.vid: v for v in variants.generate_variants(shape, variants.VariantConfig(modes=(a.mode,)),
                                                      n_images=n)}
    if a.variant not in vs:
        raise _Usage(f"unknown variant {a.variant!r}; legal: {', '.join(sorted(vs))}")
    print(_dump({"version": REPORT_VERSION, "workload": shape.name(), "variant": a.variant,
                 "launch": variants.emit_launch(vs[a.variant])},
                a.out and os.path.join(a.out, "launch.json")), end="")
    return 0


def cmd_fuse(a) -> int:
    """Alg. 3 on the first two operators of the program (heavy, element-wise, in
    either order; nests between them are the intervening code): the decision with
    its witness, the fused `.pdl` when fusable (--emit-pdl FILE or DIR/fused.pdl),
    and the executor's kernel plan (which epilogue the fused kernel applies)."""
    from . import fusion as F
    from .executor import ConvPlan, EltwisePlan, GemmPlan, plan_program
    nests = _load(a.file)
    if len(nests) < 2:
        raise _Usage("fuse needs a program of two operators")
    first_ew = not nests[0].has_kernel_call() and any(
        s.op == "=" for s in nests[0].statements()) and any(s.op == "+=" for s in nests[-1].statements())
    pair = F.OperatorPair(nests[-1], nests[0], tuple(nests[1:-1]), ew_first=True) if first_ew \
        else F.OperatorPair(nests[0], nests[-1], tuple(nests[1:-1]))
    d = F.can_fuse(pair, a.binding, strict=a.strict)
    fused_text = L.pretty(F.fuse(pair, a.binding, strict=a.strict)) if d.fusable else None
    if fused_text is not None:
        dst = a.emit_pdl or (a.out and os.path.join(a.out, "fused.pdl"))
        if dst:
            with open(dst, "w") as fh:
                fh.write(fused_text)
    plans = plan_program(nests, a.binding) if len(nests) == 2 else []
    rows = []
    for p in plans:
        kind = "conv" if isinstance(p, ConvPlan) else "gemm" if isinstance(p, GemmPlan) else "eltwise"
        ep = getattr(p, "epilogue", None)
        rows.append({"nest": p.nest, "kind": kind,
                     "fused_epilogue": None if ep is None else {
                         "nest": ep.nest, "bias": ep.bias is not None, "scale": ep.scale is not None,
                         "relu": ep.relu, "relu6": ep.relu6}})
    wit = d.witness
    print(_dump({"version": REPORT_VERSION, "file": os.path.basename(a.file),
                 "decision": {"fusable": d.fusable, "failed": d.failed, "detail": d.detail,
                              "witness": None if wit is None else json.loads(json.dumps(wit, default=list))},
                 "fused_pdl": fused_text, "plans": rows},
                a.out and os.path.join(a.out, "fusion.json")), end="")
    return 0


def cmd_train(a) -> int:
    from . import rank
    data = rank.load_dataset(a.file)
    res = rank.train_ranker(data, rank.TrainConfig(epochs=a.epochs, seed=a.seed))
    res.model.save(a.out)
    print(f"trained on {len(data)} pairs: train acc {res.train_accuracy:.3f}, "
          f"val acc {res.val_accuracy:.3f} -> {a.out}")
    return 0


def cmd_run(a) -> int:
    import numpy as np
    from .executor import interpret
    prog = L.parse_program(open(a.file).read())
    arrays, _ = interpret(prog, a.binding, seed=a.seed, mode=a.mode)
    summary = {k: {"n": int(v.size), "sum": float(np.sum(v)), "absmax": float(np.max(np.abs(v)))}
               for k, v in sorted(arrays.items())}
    print(_dump({"version": REPORT_VERSION, "mode": a.mode, "arrays": summary},
                a.out and os.path.join(a.out, "run.json")), end="")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2006_02230_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, binding=True):
        p.add_argument("file")
        if binding:
            p.add_argument("--bind", default="", help="NAME=INT,... for every parameter")
        p.add_argument("--out", default=None, help="directory for the JSON report")

    p = sub.add_parser("analyze", help="dependences + working sets (Alg. 1)")
    common(p)
    p.add_argument("--limit", type=int, default=2_000_000)
    p.set_defaults(fn=cmd_analyze)
    p = sub.add_parser("rank", help="rank tile variants and emit the top-k launch configs")
    common(p)
    p.add_argument("--method", default="both", choices=["cost", "model", "dnn", "both"])
    p.add_argument("--top-k", type=int, default=1)
    p.add_argument("--machine", default=None)
    p.add_argument("--model", default=None, help="ranker .npz (default: machines/b200_ranker.npz)")
    p.add_argument("--mode", default="3xtf32", choices=["3xtf32", "tf32"])
    p.set_defaults(fn=cmd_rank)
    p = sub.add_parser("emit", help="launch config of one variant")
    common(p)
    p.add_argument("--variant", required=True)
    p.add_argument("--mode", default="3xtf32", choices=["3xtf32", "tf32"])
    p.set_defaults(fn=cmd_emit)
    p = sub.add_parser("fuse", help="Alg. 3: can_fuse decision, fused .pdl, kernel plan")
    common(p)
    p.add_argument("--emit-pdl", default=None, help="write the fused nest here")
    p.add_argument("--strict", action="store_true",
                   help="also refuse intervening writes to the element-wise operator's inputs")
    p.set_defaults(fn=cmd_fuse)
    p = sub.add_parser("train", help="train the pairwise judge from a dataset CSV")
    p.add_argument("file")
    p.add_argument("--out", required=True)
    p.add_argument("--epochs", type=int, default=300)
    p.add_argument("--seed", type=int, default=0)
    p.set_defaults(fn=cmd_train)
    p = sub.add_parser("run", help="execute a program on the GPU (interpret drop-in)")
    common(p)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--mode", default="3xtf32", choices=["3xtf32", "tf32", "fp32"])
    p.set_defaults(fn=cmd_run)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code == 0 else 1
    try:
        if hasattr(a, "bind"):
            a.binding = _bindings(a.bind)
        if a.out and a.cmd != "train":
            os.makedirs(a.out, exist_ok=True)
        return a.fn(a)
    except _Usage as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    except L.UnboundParameterError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    except (L.ParseError, L.LoopDslError) as exc:
        print(f"parse error: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    except Exception as exc:  # analysis / ranking failure
        print(f"analysis error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 3
