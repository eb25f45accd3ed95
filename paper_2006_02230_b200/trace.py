"""Element access traces of a loop nest -- the second half of the reference's
`interpret` result (/root/reference/pkg/src/looprank/simcache.py:33-57 TraceRecord /
Trace, recorded by `run` / `eval_expr` at :146-198).

The GPU executor computes array VALUES on the B200; the trace depends only on the
nest's structure and the parameter binding, not on any value, so it is produced
here on the host by walking the IR in schedule order -- the same walk the
reference's interpreter does, without the arithmetic.  Records, in order, per
statement instance: the reads of the right-hand side in evaluation order (left
operand before right, call arguments left to right), then for `+=` a read of the
target, then the write of the target.  Schedule tuples interleave body positions
and loop counters exactly as the reference's (`sched + (pos, counter)` per loop
level, `+ (pos,)` for microkernel regions and statements); statement labels are
the nest's own or `S<i>` in preorder.

`LazyTrace` defers the walk until the records are first used: a BASELINE-sized
nest has ~1e8-1e10 records (the reference builds them eagerly, which is most of
its 7-16 us per MAC), and most drop-in callers never look at them.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, Mapping

from .loopnest import (Access, BinOp, Call, KernelCall, KernelRegion, LoopNest, LoopNode, Neg,
                       Num, StmtNode, substitute_microkernel)


class TraceError(Exception):
    """Out-of-bounds subscript or opaque kernel call while tracing."""


@dataclass(frozen=True)
class TraceRecord:
    sched: tuple     # interleaved schedule point (positions + counters)
    stmt: str
    point: tuple     # loop counter values, outermost first
    array: str
    index: int       # flattened element index
    kind: str        # "read" | "write"


@dataclass
class Trace:
    records: list

    def __len__(self) -> int:
        return len(self.records)

    def footprint(self) -> int:
        return len({(r.array, r.index) for r in self.records})

    def dump(self) -> str:
        lines = ["# trace v1: sched | stmt | point | array | index | kind"]
        for r in self.records:
            lines.append(f"{','.join(map(str, r.sched))} | {r.stmt} | "
                         f"{','.join(map(str, r.point))} | {r.array} | "
                         f"{r.index} | {r.kind}")
        return "\n".join(lines) + "\n"


class LazyTrace(Trace):
    """A Trace whose records are generated on first access."""

    def __init__(self, nest: LoopNest, binding: Mapping[str, int]):
        self._nest = nest
        self._binding = dict(binding)
        self._records = None

    @property
    def records(self) -> list:   # type: ignore[override]
        if self._records is None:
            self._records = list(iter_trace(self._nest, self._binding))
        return self._records

    def __iter__(self) -> Iterator[TraceRecord]:
        if self._records is not None:
            return iter(self._records)
        return iter_trace(self._nest, self._binding)

    def __repr__(self) -> str:
        state = "pending" if self._records is None else f"{len(self._records)} records"
        return f"LazyTrace({self._nest.name!r}, {state})"


def iter_trace(nest: LoopNest, binding: Mapping[str, int]) -> Iterator[TraceRecord]:
    """Generate the nest's access records in the reference interpreter's order."""
    if nest.has_kernel_call() and nest.microkernel is not None:
        nest = substitute_microkernel(nest)
    shapes = nest.shapes(binding)
    strides = {}
    for name, shape in shapes.items():
        st, acc = [], 1
        for extent in reversed(shape):
            st.append(acc)
            acc *= extent
        strides[name] = tuple(reversed(st))
    labels: dict = {}
    counter = [0]

    def prelabel(nodes):
        for n in nodes:
            if isinstance(n, (LoopNode, KernelRegion)):
                prelabel(n.body)
            elif isinstance(n, StmtNode):
                labels[id(n)] = n.stmt.label or f"S{counter[0]}"
                counter[0] += 1

    prelabel(nest.body)

    def flat(acc: Access, env) -> int:
        shape = shapes[acc.array]
        if len(acc.indices) != len(shape):
            raise TraceError(f"rank mismatch on {acc.array!r}")
        idx = 0
        for d, (e, extent) in enumerate(zip(acc.indices, shape)):
            v = e.eval(env)
            if not 0 <= v < extent:
                raise TraceError(f"{acc.array}[dim {d}] = {v} out of bounds [0, {extent})")
            idx += v * strides[acc.array][d]
        return idx

    def reads(expr, env, out):
        if isinstance(expr, Num):
            return
        if isinstance(expr, Neg):
            reads(expr.operand, env, out)
        elif isinstance(expr, Access):
            out.append((expr.array, flat(expr, env)))
        elif isinstance(expr, BinOp):
            reads(expr.left, env, out)
            reads(expr.right, env, out)
        elif isinstance(expr, Call):
            for a in expr.args:
                reads(a, env, out)
        else:
            raise TraceError(f"unknown expression node {expr!r}")

    env0 = {p: int(binding[p]) for p in nest.params}

    def run(nodes, env, sched, point):
        for pos, n in enumerate(nodes):
            if isinstance(n, LoopNode):
                lp = n.loop
                value = lp.lower.eval(env)
                hi = min(u.eval(env) for u in lp.upper)
                cnt = 0
                while value < hi:
                    yield from run(n.body, {**env, lp.iterator: value}, sched + (pos, cnt), point + (cnt,))
                    value += lp.step
                    cnt += 1
            elif isinstance(n, KernelRegion):
                yield from run(n.body, env, sched + (pos,), point)
            elif isinstance(n, StmtNode):
                stmt = n.stmt
                label = labels[id(n)]
                s = sched + (pos,)
                rd: list = []
                reads(stmt.expr, env, rd)
                for arr, i in rd:
                    yield TraceRecord(s, label, point, arr, i, "read")
                i = flat(stmt.target, env)
                if stmt.op == "+=":
                    yield TraceRecord(s, label, point, stmt.target.array, i, "read")
                yield TraceRecord(s, label, point, stmt.target.array, i, "write")
            elif isinstance(n, KernelCall):
                raise TraceError(f"cannot trace opaque kernel call {n!r}; substitute first")
            else:
                raise TraceError(f"unknown node {n!r}")

    yield from run(nest.body, env0, (), ())
