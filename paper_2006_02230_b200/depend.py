"""Polyhedral front end of the ranker, evaluated at bound parameters.

Mirrors the reference's analysis entry points with the same names and
results, computed by exact enumeration of the bound nest instead of a
symbolic integer-set engine (the reference spends 88% of its analysis time in
emptiness tests; enumeration is exact at the desk-size bindings
the analysis runs on and takes milliseconds):

  extract_polyhedral  (loopdsl.py:837-905)  -> PolyInfo / StmtInfo / RefInfo
  compute_dependences (depend.py:109-125)   -> one Dependence per ordered pair of
                                              references to an array with a
                                              same-element, strictly-later pair
  classify_parallel_span (depend.py:128-159) -> whether source and target can
                                              differ in a shared parallel iterator
  domain_size / domain_lexmin / domain_lexmax (polyset.py IntSet.cardinality
                                              753-771, lexmin/lexmax 718-732)

Dependence ids are "<src ref>-><tgt ref>" with ref ids "<stmt>:r<k>" (reads in
textual order, a `+=` target read last) and "<stmt>:w0", as in the reference.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Mapping

from .loopnest import KernelRegion, LoopNest, LoopNode, StmtNode, substitute_microkernel
from .wset import _KIND, _Trace


@dataclass(frozen=True)
class RefInfo:
    ref_id: str
    stmt_label: str
    array: str
    kind: str            # "read" | "write"
    index_exprs: tuple   # loopnest.Affine subscripts


@dataclass(frozen=True)
class StmtInfo:
    label: str
    loop_iters: tuple
    parallel_iters: tuple
    reads: tuple
    writes: tuple

    def refs(self) -> tuple:
        return self.reads + self.writes


@dataclass(frozen=True)
class PolyInfo:
    nest: LoopNest
    statements: tuple

    def statement(self, label: str) -> StmtInfo:
        for s in self.statements:
            if s.label == label:
                return s
        raise KeyError(label)

    def all_refs(self) -> list:
        return [r for s in self.statements for r in s.refs()]


@dataclass(frozen=True)
class Dependence:
    kind: str
    array: str
    source_ref: str
    target_ref: str
    source_stmt: str
    target_stmt: str
    spans_parallel: bool = False
    parallel_iterator: str | None = None

    @property
    def dep_id(self) -> str:
        return f"{self.source_ref}->{self.target_ref}"


def extract_polyhedral(nest: LoopNest) -> PolyInfo:
    if nest.has_kernel_call():
        nest = substitute_microkernel(nest)
    stmts, auto = [], [0]

    def walk(nodes, iters, pars):
        for n in nodes:
            if isinstance(n, LoopNode):
                it = n.loop.iterator
                walk(n.body, iters + (it,), pars + ((it,) if n.loop.parallel else ()))
            elif isinstance(n, KernelRegion):
                walk(n.body, iters, pars)
            elif isinstance(n, StmtNode):
                st = n.stmt
                label = st.label or f"S{auto[0]}"
                auto[0] += 1
                reads = tuple(RefInfo(f"{label}:r{k}", label, a.array, "read", tuple(a.indices))
                              for k, a in enumerate(st.read_accesses()))
                writes = (RefInfo(f"{label}:w0", label, st.target.array, "write",
                                  tuple(st.target.indices)),)
                stmts.append(StmtInfo(label, iters, pars, reads, writes))

    walk(nest.body, (), ())
    return PolyInfo(nest, tuple(stmts))


class _Bound:
    """The enumerated nest under one binding (cached per (nest, binding))."""
    _cache: dict = {}

    @classmethod
    def of(cls, info: PolyInfo, binding: Mapping[str, int]):
        key = (id(info.nest), tuple(sorted(binding.items())))
        hit = cls._cache.get(key)
        if hit is None or hit[0] is not info.nest:
            tr = _Trace(info.nest, binding, 2_000_000)
            pos = {rid: {} for rid in tr.refs}
            for i, (_, _, elems) in enumerate(tr.inst):
                for rid, e in elems.items():
                    pos[rid].setdefault(e, []).append(i)
            hit = (info.nest, tr, pos)
            if len(cls._cache) > 32:
                cls._cache.clear()
            cls._cache[key] = hit
        return hit[1], hit[2]


def compute_dependences(info: PolyInfo, binding: Mapping[str, int]) -> list:
    """Every ordered reference pair on one array with at least one
    (source, strictly later target) instance pair touching the same element."""
    tr, pos = _Bound.of(info, binding)
    refs = [r for s in info.statements for r in s.refs()]
    out = []
    for src in refs:
        for tgt in refs:
            if src.array != tgt.array:
                continue
            found = False
            for e, s_list in pos[src.ref_id].items():
                t_list = pos[tgt.ref_id].get(e)
                if t_list and max(t_list) > min(s_list):
                    found = True
                    break
            if found:
                out.append(Dependence(_KIND[(src.kind, tgt.kind)], src.array, src.ref_id, tgt.ref_id,
                                      src.stmt_label, tgt.stmt_label))
    return out


def classify_parallel_span(dep: Dependence, info: PolyInfo,
                           binding: Mapping[str, int]) -> Dependence:
    """spans_parallel iff some dependent instance pair differs in a parallel
    iterator enclosing both statements (exact under the binding)."""
    s_st, t_st = info.statement(dep.source_stmt), info.statement(dep.target_stmt)
    common = [p for p in s_st.parallel_iters if p in t_st.parallel_iters]
    if not common:
        return replace(dep, spans_parallel=False, parallel_iterator=None)
    tr, pos = _Bound.of(info, binding)
    for p in common:
        ps, pt = s_st.loop_iters.index(p), t_st.loop_iters.index(p)
        for e, s_list in pos[dep.source_ref].items():
            t_list = pos[dep.target_ref].get(e, ())
            for i in s_list:
                ci = tr.inst[i][1][ps]
                for t in t_list:
                    if t > i and tr.inst[t][1][pt] != ci:
                        return replace(dep, spans_parallel=True,
                                       parallel_iterator=s_st.parallel_iters[0])
    return replace(dep, spans_parallel=False, parallel_iterator=None)


def _points(info: PolyInfo, label: str, binding: Mapping[str, int]) -> list:
    tr, _ = _Bound.of(info, binding)
    iters = info.statement(label).loop_iters
    return [tuple(ctr) for (lab, ctr, _) in tr.inst if lab == label], iters


def domain_size(info: PolyInfo, label: str, binding: Mapping[str, int]) -> int:
    """Number of instances of statement `label` (IntSet.cardinality)."""
    pts, _ = _points(info, label, binding)
    return len(pts)


def domain_lexmin(info: PolyInfo, label: str, binding: Mapping[str, int]):
    """Lexicographically first instance as {iterator: value} (trip counter for
    non-unit-step loops), None if empty."""
    return _extreme(info, label, binding, min)


def domain_lexmax(info: PolyInfo, label: str, binding: Mapping[str, int]):
    return _extreme(info, label, binding, max)


def _extreme(info, label, binding, pick):
    tr, _ = _Bound.of(info, binding)
    inst = [(ctr, elems) for (lab, ctr, elems) in tr.inst if lab == label]
    if not inst:
        return None
    ctr = pick(c for c, _ in inst)
    # recover iterator values by replaying the loop bounds for these trip counters
    return _iter_values(info, label, binding, ctr)


def _iter_values(info, label, binding, ctr):
    from .loopnest import Loop  # noqa: F401  (type only)
    env = {p: int(binding[p]) for p in info.nest.params}
    vals = {}
    nodes = info.nest.body
    for depth, it in enumerate(info.statement(label).loop_iters):
        node = _find_loop(nodes, it)
        lo = node.loop.lower.eval(env)
        v = lo + ctr[depth] * node.loop.step
        env[it] = v
        # non-unit steps are normalised to the trip counter, as the reference's
        # extract_polyhedral does (loopdsl.py:860-865)
        vals[it] = v if node.loop.step == 1 else ctr[depth]
        nodes = node.body
    return vals


def _find_loop(nodes, it):
    for n in nodes:
        if isinstance(n, LoopNode):
            if n.loop.iterator == it:
                return n
            hit = _find_loop(n.body, it)
            if hit is not None:
                return hit
        elif isinstance(n, KernelRegion):
            hit = _find_loop(n.body, it)
            if hit is not None:
                return hit
    return None
