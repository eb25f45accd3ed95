"""Alg. 3 operator fusion on the loop-nest IR.

A compute-heavy nest (conv, GEMM) and an adjacent element-wise nest over its
output (bias + ReLU, ReLU6, batch-norm inference affine) are fused by inserting
the element-wise statement into the LAST iteration of the heavy nest's
reduction loops, which index-set splitting peels off the main loop (§5).  The
peeled form is what the B200 kernels implement as their fused epilogue: the
element-wise op runs on each output value once its reduction is complete
(csrc/pdl_kernels.cuh `epilogue4`, flags PDL_BIAS / PDL_RELU / PDL_RELU6 /
PDL_SCALE).

* `write_set(nest, b)`     per-array set of elements the nest writes (Alg. 3 line 1)
* `can_fuse(pair, b)`      Alg. 3 lines 4-6, checked in order, first failure with a
                           witness: (1) W_hy = W_ew; (2) |I_ew| = |W_ew| and the
                           element-wise statement reads the write set only at the
                           element it writes; (3) no intervening statement reads or
                           writes an element of W_hy.  Structural preconditions of the
                           peel (ledger below) are reported as `not-invertible` /
                           `non-rectangular-reduction`.
* `fuse(pair, b)`          the fused LoopNest: main reduction ranges minus the last
                           iteration, the peeled copy with the element-wise statement
                           right after the heavy one (or, for an element-wise nest
                           that PRECEDES the heavy one, the peeled FIRST iteration with
                           the element-wise statement before it).  No guards in the
                           hot loop; reduction extent 1 leaves an empty main loop.
                           A `FusedNest` remembers its pair so the GPU executor can
                           map it onto the fused kernel.

Condition checks enumerate the iteration spaces under the concrete binding
(SPEC: "set equalities via cardinality + containment"), so they are meant for
desk-sized bindings; the executor's plan_program applies the same three
conditions structurally to nests it has matched as conv / GEMM / element-wise.

Paper-gap ledger: the element-wise iterators must be an
invertible affine image of the heavy nest's output iterators (each element-wise
iterator in exactly one output subscript, coefficient +-1); the heavy nest's
reduction loops (iterators absent from its write subscripts) must have constant
bounds (parameters only), a single upper bound and step 1; both nests hold one
statement each.  Intervening nests (condition 3 holds) are returned by the
caller after the fused nest; `strict=True` also refuses intervening writes to
arrays the element-wise statement reads (SPEC Open Question).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Iterator, Mapping

from .loopnest import (Access, Affine, BinOp, Call, KernelRegion, LoopDslError, LoopNest,
                       LoopNode, Neg, Num, Statement, StmtNode, UnboundParameterError,
                       expr_accesses, statements_with_loops, substitute_microkernel, walk)

__all__ = ["OperatorPair", "FusionDecision", "FusedNest", "FusionError", "write_set", "can_fuse",
           "fuse", "WRITE_SETS_DIFFER", "NOT_ELEMENTWISE", "INTERVENING_ACCESS", "NOT_INVERTIBLE",
           "NON_RECTANGULAR"]

WRITE_SETS_DIFFER = "write-sets-differ"
NOT_ELEMENTWISE = "not-elementwise"
INTERVENING_ACCESS = "intervening-access"
NOT_INVERTIBLE = "not-invertible"
NON_RECTANGULAR = "non-rectangular-reduction"


class FusionError(LoopDslError):
    """fuse() precondition violated (carries the FusionDecision)."""

    def __init__(self, decision: "FusionDecision"):
        super().__init__(f"not fusable: {decision.failed} ({decision.detail})")
        self.decision = decision


@dataclass(frozen=True)
class OperatorPair:
    """Alg. 3 inputs: heavy nest op_hy, element-wise nest op_ew, the nests between
    them (possibly none) and which comes first in program order."""
    heavy: LoopNest
    eltwise: LoopNest
    between: tuple = ()
    ew_first: bool = False


@dataclass(frozen=True)
class FusionDecision:
    fusable: bool
    failed: str | None = None
    witness: object = None
    detail: str = ""


@dataclass(frozen=True)
class FusedNest(LoopNest):
    """A fused nest (a LoopNest: prints, parses back and interprets like one) that
    remembers the operator pair it came from."""
    pair: OperatorPair | None = field(default=None, compare=False)


# ----------------------------------------------------------------------------- enumeration
def _prep(nest: LoopNest) -> LoopNest:
    return substitute_microkernel(nest) if nest.has_kernel_call() else nest


def _env0(nest: LoopNest, binding: Mapping[str, int]) -> dict:
    missing = [p for p in nest.params if p not in binding]
    if missing:
        raise UnboundParameterError(f"unbound parameters: {missing}")
    return {p: int(binding[p]) for p in nest.params}


def _instances(nest: LoopNest, binding) -> Iterator[tuple]:
    """(statement, env) for every statement instance, in schedule order (env is
    reused between yields: copy what you keep)."""
    env = _env0(nest, binding)

    def run(nodes):
        for n in nodes:
            if isinstance(n, LoopNode):
                lp = n.loop
                v = lp.lower.eval(env)
                hi = min(u.eval(env) for u in lp.upper)
                while v < hi:
                    env[lp.iterator] = v
                    yield from run(n.body)
                    v += lp.step
                env.pop(lp.iterator, None)
            elif isinstance(n, KernelRegion):
                yield from run(n.body)
            elif isinstance(n, StmtNode):
                yield n.stmt, env

    yield from run(_prep(nest).body)


def _elem(acc: Access, env) -> tuple:
    return tuple(ix.eval(env) for ix in acc.indices)


def _accesses(stmt: Statement) -> list:
    """(access, is_write) of one statement instance, reads first."""
    return [(a, False) for a in stmt.read_accesses()] + [(stmt.target, True)]


def write_set(nest: LoopNest, binding: Mapping[str, int]) -> dict:
    """{array: frozenset of element index tuples} written by the nest (the union of
    the images of its write relations over the iteration space)."""
    out: dict = {}
    for stmt, env in _instances(nest, binding):
        out.setdefault(stmt.target.array, set()).add(_elem(stmt.target, env))
    return {a: frozenset(s) for a, s in out.items()}


# ----------------------------------------------------------------------------- structure
def _single(nest: LoopNest) -> tuple:
    sl = list(statements_with_loops(_prep(nest).body))
    if len(sl) != 1:
        return None, None
    return sl[0]


def _ew_to_hy(ew_stmt: Statement, hy_stmt: Statement, ew_loops) -> dict | None:
    """Element-wise iterator -> affine form over the heavy nest's iterators, read off
    the two write subscripts (None if the correspondence is not invertible)."""
    ew_iters = {lp.iterator for lp in ew_loops}
    if len(ew_stmt.target.indices) != len(hy_stmt.target.indices):
        return None
    sol: dict = {}
    for e, h in zip(ew_stmt.target.indices, hy_stmt.target.indices):
        its = [v for v in e.variables() if v in ew_iters]
        if len(its) > 1:
            return None
        if not its:
            continue
        it = its[0]
        c = e.coeff(it)
        if abs(c) != 1 or it in sol:
            return None
        rest = e - Affine({it: c})
        sol[it] = (h - rest).scale(c)
    if set(sol) != ew_iters:
        return None
    return sol


def _reduction_loops(hy_stmt: Statement, hy_loops) -> list | None:
    written = set()
    for ix in hy_stmt.target.indices:
        written |= ix.variables()
    red = [lp for lp in hy_loops if lp.iterator not in written]
    iters = {lp.iterator for lp in hy_loops}
    for lp in red:
        if lp.step != 1 or len(lp.upper) != 1:
            return None
        if (lp.lower.variables() | lp.upper[0].variables()) & iters:
            return None
    return red


# ----------------------------------------------------------------------------- Alg. 3 checks
def can_fuse(pair: OperatorPair, binding: Mapping[str, int], strict: bool = False) -> FusionDecision:
    """Alg. 3 lines 4-6 under `binding`: first failed condition with a witness."""
    hy, ew = _prep(pair.heavy), _prep(pair.eltwise)
    w_hy, w_ew = write_set(hy, binding), write_set(ew, binding)
    # (1) same elements
    if set(w_hy) != set(w_ew):
        arr = sorted(set(w_hy) ^ set(w_ew))[0]
        return FusionDecision(False, WRITE_SETS_DIFFER, (arr, None),
                              f"array {arr!r} written by only one operator")
    for arr in sorted(w_hy):
        diff = w_hy[arr] ^ w_ew[arr]
        if diff:
            el = min(diff)
            who = "heavy" if el in w_hy[arr] else "element-wise"
            return FusionDecision(False, WRITE_SETS_DIFFER, (arr, el),
                                  f"{arr}{list(el)} written only by the {who} operator")
    # (2) element-wise: one instance per element, no reduction, reads W only at its own element
    n_inst = 0
    seen: set = set()
    for stmt, env in _instances(ew, binding):
        n_inst += 1
        el = _elem(stmt.target, env)
        if stmt.op != "=":
            return FusionDecision(False, NOT_ELEMENTWISE, (stmt.target.array, el),
                                  f"'{stmt.op}' accumulates: a reduction, not element-wise")
        if (stmt.target.array, el) in seen:
            return FusionDecision(False, NOT_ELEMENTWISE, (stmt.target.array, el),
                                  f"|I_ew| > |W_ew|: {stmt.target.array}{list(el)} written twice")
        seen.add((stmt.target.array, el))
        for acc in expr_accesses(stmt.expr):
            if acc.array in w_hy:
                rel = _elem(acc, env)
                if acc.array != stmt.target.array or rel != el:
                    return FusionDecision(False, NOT_ELEMENTWISE, (acc.array, rel),
                                          f"reads {acc.array}{list(rel)} while writing "
                                          f"{stmt.target.array}{list(el)}")
    if n_inst != sum(len(s) for s in w_ew.values()):
        return FusionDecision(False, NOT_ELEMENTWISE, n_inst, "|I_ew| != |W_ew|")
    # (3) nothing in between touches W_hy (strict: nor writes what op_ew reads)
    ew_reads = {a.array for s in ew.statements() for a in expr_accesses(s.expr)}
    for mid in pair.between:
        for stmt, env in _instances(mid, binding):
            for acc, is_w in _accesses(stmt):
                el = _elem(acc, env)
                if acc.array in w_hy and el in w_hy[acc.array]:
                    return FusionDecision(False, INTERVENING_ACCESS,
                                          (mid.name, stmt.label, acc.array, el),
                                          f"{mid.name}:{stmt.label or '?'} "
                                          f"{'writes' if is_w else 'reads'} {acc.array}{list(el)}")
                if strict and is_w and acc.array in ew_reads:
                    return FusionDecision(False, INTERVENING_ACCESS,
                                          (mid.name, stmt.label, acc.array, el),
                                          f"{mid.name}:{stmt.label or '?'} writes {acc.array}"
                                          f"{list(el)}, an input of the element-wise operator")
    # structural preconditions of the peel
    hs, hl = _single(hy)
    es, el_ = _single(ew)
    if hs is None or es is None:
        return FusionDecision(False, NOT_INVERTIBLE, None, "each operator must be one statement")
    for acc in hs.read_accesses():
        if acc.array in w_hy and acc != replace(hs.target, kind="read"):
            return FusionDecision(False, NOT_ELEMENTWISE, (acc.array, None),
                                  "the heavy operator reads its own write set off its target")
    if _ew_to_hy(es, hs, el_) is None:
        return FusionDecision(False, NOT_INVERTIBLE, None,
                              "element-wise iterators are not an invertible image of the "
                              "heavy operator's output iterators")
    if _reduction_loops(hs, hl) is None:
        return FusionDecision(False, NON_RECTANGULAR, None,
                              "reduction loops need constant bounds, one upper bound, step 1")
    return FusionDecision(True)


# ----------------------------------------------------------------------------- the transformation
def _subst_expr(e, env):
    if isinstance(e, Access):
        return replace(e, indices=tuple(ix.subst(env) for ix in e.indices))
    if isinstance(e, BinOp):
        return BinOp(e.op, _subst_expr(e.left, env), _subst_expr(e.right, env))
    if isinstance(e, Neg):
        return Neg(_subst_expr(e.operand, env))
    if isinstance(e, Call):
        return Call(e.fn, tuple(_subst_expr(a, env) for a in e.args))
    return e


def _subst_stmt(s: Statement, env, label=None) -> Statement:
    return Statement(s.label if label is None else label, _subst_expr(s.target, env), s.op,
                     _subst_expr(s.expr, env))


def _subst_nodes(nodes, env) -> tuple:
    out = []
    for n in nodes:
        if isinstance(n, LoopNode):
            lp = n.loop
            lp2 = replace(lp, lower=lp.lower.subst(env), upper=tuple(u.subst(env) for u in lp.upper))
            out.append(LoopNode(lp2, _subst_nodes(n.body, env)))
        elif isinstance(n, KernelRegion):
            out.extend(_subst_nodes(n.body, env))     # the band is no longer the microkernel's
        elif isinstance(n, StmtNode):
            out.append(StmtNode(_subst_stmt(n.stmt, env)))
        else:
            out.append(n)
    return tuple(out)


def fuse(pair: OperatorPair, binding: Mapping[str, int], strict: bool = False) -> FusedNest:
    """The fused nest (Alg. 3 lines 8-10).  Raises FusionError when can_fuse fails
    (the caller keeps the original pair, Alg. 3 lines 12-14)."""
    d = can_fuse(pair, binding, strict)
    if not d.fusable:
        raise FusionError(d)
    hy, ew = _prep(pair.heavy), _prep(pair.eltwise)
    hs, hl = _single(hy)
    es, el_ = _single(ew)
    ew_stmt = _subst_stmt(es, _ew_to_hy(es, hs, el_))
    red = {lp.iterator for lp in _reduction_loops(hs, hl)}

    def peel(nodes) -> tuple:
        out = []
        for n in nodes:
            if isinstance(n, LoopNode) and n.loop.iterator in red:
                lp = n.loop
                body = _subst_nodes(n.body, {})            # flattens marked bands
                if pair.ew_first:
                    first = _subst_nodes(body, {lp.iterator: lp.lower})
                    out.extend(peel(first))
                    out.append(LoopNode(replace(lp, lower=lp.lower + 1), body))
                else:
                    out.append(LoopNode(replace(lp, upper=(lp.upper[0] - 1,)), body))
                    out.extend(peel(_subst_nodes(body, {lp.iterator: lp.upper[0] - 1})))
            elif isinstance(n, LoopNode):
                out.append(LoopNode(n.loop, peel(n.body)))
            elif isinstance(n, KernelRegion):
                out.extend(peel(n.body))
            elif isinstance(n, StmtNode) and n.stmt.target.array == hs.target.array:
                # every reduction loop on the path is at its last (first) iteration here
                s = n.stmt
                if pair.ew_first:
                    out += [StmtNode(ew_stmt), StmtNode(s)]
                else:
                    out += [StmtNode(s), StmtNode(ew_stmt)]
            else:
                out.append(n)
        return tuple(out)

    # the heavy statement now has one copy per peel level: distinct labels (the
    # polyhedral extraction keys statements by label)
    seen = [0]

    def relabel(nodes) -> tuple:
        out = []
        for n in nodes:
            if isinstance(n, LoopNode):
                n = LoopNode(n.loop, relabel(n.body))
            elif isinstance(n, StmtNode) and n.stmt.label and n.stmt.label == hs.label:
                if seen[0]:
                    n = StmtNode(replace(n.stmt, label=f"{hs.label}_p{seen[0]}"))
                seen[0] += 1
            out.append(n)
        return tuple(out)

    body = relabel(peel(hy.body))
    arrays = dict(hy.arrays)
    for a, dims in ew.arrays:
        arrays.setdefault(a, dims)
    params = tuple(dict.fromkeys(hy.params + ew.params))
    name = f"{hy.name}_{ew.name}" if hy.name and ew.name else (hy.name or ew.name)
    return FusedNest(name=name, params=params, arrays=tuple(arrays.items()), body=body,
                     microkernel=None, pair=pair)
