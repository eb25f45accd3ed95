"""Pure-Python interpreter of the loop-nest IR -- TEST INFRASTRUCTURE (small cases).

A restatement of the reference's `looprank.simcache.interpret`
(/root/reference/pkg/src/looprank/simcache.py:89-204) over this repo's IR
(paper_2006_02230_b200.loopnest): float64 arrays, statements executed in
schedule order, `+=` as `a[i] = a[i] + value` with the value computed first,
`min` / `max` with Python's semantics (the first minimal / maximal argument
wins, so max(-0.0, 0.0) keeps -0.0), every subscript bounds-checked.  No trace.

It exists to check IR transformations on the CPU -- the Alg. 3 fusion pass
(paper_2006_02230_b200.fusion) must leave every output bit unchanged -- and is
pinned against the reference's own outputs (tests/golden/conv_*_relu.npz, made
by running the unmodified reference interpreter).  Sizes: up to ~1e6 statement
instances (a few seconds).
"""
from __future__ import annotations

from typing import Mapping

import numpy as np

from paper_2006_02230_b200.loopnest import (Access, BinOp, Call, KernelCall, KernelRegion,
                                            LoopNest, LoopNode, Neg, Num, Program, StmtNode,
                                            UnboundParameterError, substitute_microkernel)


class OracleInterpError(Exception):
    pass


def _compile_access(acc: Access, shapes, env0):
    """(array, per-dim [(c0, ((iter, coef), ...), extent)], strides) with the
    parameters folded into c0."""
    shape = shapes[acc.array]
    if len(acc.indices) != len(shape):
        raise OracleInterpError(f"rank mismatch on {acc.array!r}")
    dims = []
    for e, extent in zip(acc.indices, shape):
        c0 = e.c0
        terms = []
        for name, c in e.terms.items():
            if name in env0:
                c0 += c * env0[name]
            else:
                terms.append((name, c))
        dims.append((c0, tuple(terms), extent))
    strides = []
    acc_s = 1
    for extent in reversed(shape):
        strides.append(acc_s)
        acc_s *= extent
    return acc.array, tuple(dims), tuple(reversed(strides))


def interpret(nest, binding: Mapping[str, int], inputs: Mapping[str, np.ndarray]) -> dict:
    """Run a LoopNest (or every nest of a Program, in order) on float64 copies of
    `inputs`; returns {array: flat float64 ndarray}."""
    nests = list(nest.nests) if isinstance(nest, Program) else [nest]
    arrays = {k: np.array(v, dtype=np.float64).ravel() for k, v in inputs.items()}
    for n in nests:
        _run_nest(n, binding, arrays)
    return arrays


def _run_nest(nest: LoopNest, binding, arrays) -> None:
    if nest.has_kernel_call() and nest.microkernel is not None:
        nest = substitute_microkernel(nest)
    missing = [p for p in nest.params if p not in binding]
    if missing:
        raise UnboundParameterError(f"unbound parameters: {missing}")
    shapes = nest.shapes(binding)
    for name, shape in shapes.items():
        need = int(np.prod(shape)) if shape else 1
        if name not in arrays or arrays[name].size < need:
            raise OracleInterpError(f"input array {name!r} too small")
    env0 = {p: int(binding[p]) for p in nest.params}
    cache: dict = {}

    def flat(acc: Access, env) -> int:
        key = id(acc)
        comp = cache.get(key)
        if comp is None:
            comp = cache[key] = (acc, _compile_access(acc, shapes, env0))
        _, (_, dims, strides) = comp
        idx = 0
        for d, ((c0, terms, extent), st) in enumerate(zip(dims, strides)):
            v = c0
            for name, c in terms:
                v += c * env[name]
            if not 0 <= v < extent:
                raise OracleInterpError(f"{acc.array}[dim {d}] = {v} out of bounds [0, {extent})")
            idx += v * st
        return idx

    def ev(e, env) -> float:
        if isinstance(e, Num):
            return e.value
        if isinstance(e, Access):
            return arrays[e.array][flat(e, env)]
        if isinstance(e, BinOp):
            a = ev(e.left, env)
            b = ev(e.right, env)
            if e.op == "+":
                return a + b
            if e.op == "-":
                return a - b
            if e.op == "*":
                return a * b
            return a / b
        if isinstance(e, Neg):
            return -ev(e.operand, env)
        if isinstance(e, Call):
            vals = [ev(a, env) for a in e.args]
            return min(vals) if e.fn == "min" else max(vals)
        raise OracleInterpError(f"unknown expression node {e!r}")

    def run(nodes, env) -> None:
        for n in nodes:
            if isinstance(n, LoopNode):
                lp = n.loop
                v = lp.lower.eval(env)
                hi = min(u.eval(env) for u in lp.upper)
                while v < hi:
                    env[lp.iterator] = v
                    run(n.body, env)
                    v += lp.step
                env.pop(lp.iterator, None)
            elif isinstance(n, KernelRegion):
                run(n.body, env)
            elif isinstance(n, StmtNode):
                s = n.stmt
                value = ev(s.expr, env)
                i = flat(s.target, env)
                arr = arrays[s.target.array]
                if s.op == "+=":
                    arr[i] = arr[i] + value
                else:
                    arr[i] = value
            elif isinstance(n, KernelCall):
                raise OracleInterpError(f"opaque kernel call {n.name!r}; substitute first")
            else:
                raise OracleInterpError(f"unknown node {n!r}")

    run(nest.body, dict(env0))
