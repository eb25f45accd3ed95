"""GPU executor behind the reference's `interpret` entry point.

`interpret(nest, binding, inputs=...)` mirrors `looprank.simcache.interpret`
(/root/reference/pkg/src/looprank/simcache.py:89-204): it takes a parsed
`LoopNest` (or a `Program` of several nests sharing arrays), a parameter
binding and a dict of input arrays, and returns the final contents of every
array as flat float64 numpy arrays.  Instead of walking the iteration space
element by element it recognises the nests the PolyDL hot path consists of and
launches the B200 kernels:

* the Fig. 9 blocked convolution -- any loop order, tiling
  or parallel marking of it, with or without the `#pragma microkernel` band;
* the Fig. 1 / Fig. 12 GEMM;
* an element-wise epilogue nest over the conv / GEMM output: an optional
  per-channel scale (batch-norm inference affine `y * s[k]`), an optional bias /
  shift `+ b[k]`, then optionally ReLU `max(., 0.0)` or ReLU6
  `min(max(., 0.0), 6.0)`.  It is fused into the preceding
  heavy nest when Alg. 3's conditions hold:
  same write set, element-wise, nothing in between -- the kernels then apply it
  in their epilogue (PDL_SCALE / PDL_BIAS / PDL_RELU / PDL_RELU6);
* a `fusion.FusedNest` (the output of `fusion.fuse`), executed as its operator
  pair with the element-wise part in the kernel epilogue.

Recognition is semantic, not textual: every array subscript is an affine form
over the loop iterators; the executor assigns the iterators to the roles of the
contraction (image, output-channel tile, ..., reduction lanes), checks that
each role is a mixed-radix combination of disjoint iterators (so the map from
iteration points to index tuples is injective) and that the iteration count
equals the size of the index space (so it is onto).  A nest that is not one of
these raises `InterpreterError` -- there is no CPU fallback.

Semantics kept from the reference: `+=` accumulates into the array's incoming
contents; arrays not written are returned unchanged; parameters must all be
bound (`UnboundParameterError`); missing / short inputs raise.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .loopnest import (Access, Affine, BinOp, Call, LoopNest, Num, Program, StmtNode,
                       UnboundParameterError, statements_with_loops, substitute_microkernel,
                       walk, KernelCall)

__all__ = ["InterpreterError", "UnboundParameterError", "interpret", "execute", "plan_program",
           "make_inputs", "ConvPlan", "GemmPlan", "EltwisePlan"]


class InterpreterError(Exception):
    """The nest cannot be executed (unsupported shape, bad inputs, opaque call)."""


# ----------------------------------------------------------------------------- plans
@dataclass
class ConvPlan:
    nest: str
    out: str
    filt: str
    inp: str
    N: int
    KT: int
    CT: int
    P: int
    Q: int
    R: int
    S: int
    stride: int
    Hp: int
    Wp: int
    parallel_role: str | None = None       # role of the outermost parallel loop (sharding axis)
    epilogue: "EltwisePlan | None" = None

    @property
    def flops(self) -> float:
        return 2.0 * self.N * self.KT * 16 * self.CT * 16 * self.R * self.S * self.P * self.Q


@dataclass
class GemmPlan:
    nest: str
    C: str
    A: str
    B: str
    M: int
    N: int
    K: int
    parallel_role: str | None = None
    epilogue: "EltwisePlan | None" = None

    @property
    def flops(self) -> float:
        return 2.0 * self.M * self.N * self.K


@dataclass
class EltwisePlan:
    nest: str
    target: str
    bias: str | None
    relu: bool
    relu6: bool
    bias_axes: tuple = ()   # target dims the bias is indexed by
    scale: str | None = None
    scale_axes: tuple = ()  # target dims the scale is indexed by

    def channel_axes_ok(self, axes: tuple) -> bool:
        """bias / scale indexed exactly by the output-channel dims `axes`."""
        return (self.bias is None or self.bias_axes == axes) and \
            (self.scale is None or self.scale_axes == axes)


# ----------------------------------------------------------------------------- helpers
def _loop_ranges(loops, env) -> dict:
    """Iterator -> (min, max, step) over the whole domain (bounds may depend on
    outer iterators; affine bounds are monotone, so the corners suffice)."""
    rng: dict = {}
    for lp in loops:
        corners = [{**env, **{k: v[0] for k, v in rng.items()}},
                   {**env, **{k: v[1] for k, v in rng.items()}}]
        lo = min(lp.lower.eval(c) for c in corners)
        hi = max(min(u.eval(c) for u in lp.upper) for c in corners) - 1
        if hi < lo:
            rng[lp.iterator] = (lo, lo - 1, lp.step)
        else:
            rng[lp.iterator] = (lo, lo + ((hi - lo) // lp.step) * lp.step, lp.step)
    return rng


def _count(loops, env) -> int:
    """Exact number of iteration points of a perfect loop band (outer-to-inner)."""
    if not loops:
        return 1
    lp, rest = loops[0], loops[1:]
    dependent = any(lp.iterator in u.variables() or lp.iterator in r.lower.variables()
                    for r in rest for u in r.upper)
    if not dependent:
        return lp.trip_count(env) * _count(rest, env)
    total = 0
    lo = lp.lower.eval(env)
    hi = min(u.eval(env) for u in lp.upper)
    for v in range(lo, hi, lp.step):
        total += _count(rest, {**env, lp.iterator: v})
    return total


def _role_ok(expr: Affine, ranges: Mapping[str, tuple], extent: int, iters: set) -> bool:
    """expr is an injective mixed-radix form over loop iterators covering [0, extent)."""
    its = [n for n in expr.terms if n in iters]
    if any(n not in iters for n in expr.terms):
        return False          # depends on a parameter: not a plain index
    if not its:
        return extent == 1 and expr.c0 == 0
    # iterator v = lo + step*u, u in [0, trips): digit weight c*step, digit range trips
    parts = []
    base = expr.c0
    for n in its:
        c = expr.terms[n]
        lo, hi, step = ranges[n]
        if c <= 0 or hi < lo:
            return False
        parts.append((c * step, (hi - lo) // step))
        base += c * lo
    if base != 0:
        return False
    parts.sort()
    reach = 0
    for w, umax in parts:
        if w <= reach:                 # overlaps the lower digits: not injective
            return False
        reach += w * umax
    return reach < extent              # image inside [0, extent); onto via the count check


def _single_stmt(nest: LoopNest):
    items = list(statements_with_loops(nest.body))
    if len(items) != 1:
        raise InterpreterError(f"nest {nest.name!r}: expected one statement, found {len(items)}")
    return items[0]


def _product_operands(expr):
    if isinstance(expr, BinOp) and expr.op == "*" and isinstance(expr.left, Access) \
            and isinstance(expr.right, Access):
        return expr.left, expr.right
    return None


# ----------------------------------------------------------------------------- recognisers
def _match_conv(nest, stmt, loops, env, shapes):
    ops = _product_operands(stmt.expr)
    tgt = stmt.target
    if stmt.op != "+=" or ops is None or len(tgt.indices) != 5:
        return None
    a, b = ops
    filt, inp = (a, b) if len(a.indices) == 6 else (b, a)
    if len(filt.indices) != 6 or len(inp.indices) != 5:
        return None
    o, f, x = tgt.indices, filt.indices, inp.indices
    img, kt, oj, oi, ofm = o
    if not (x[0] == img and f[0] == kt and f[5] == ofm and f[1] == x[1] and f[4] == x[4]):
        return None
    ct, kj, ki, ifm = f[1], f[2], f[3], f[4]
    stride = None
    for s in (1, 2, 3, 4):
        if x[2] == oj.scale(s) + kj and x[3] == oi.scale(s) + ki:
            stride = s
            break
    if stride is None:
        return None
    so, sf, sx = shapes[tgt.array], shapes[filt.array], shapes[inp.array]
    N, KT, P, Q, V = so
    KT2, CT, R, S, C16, K16 = sf
    N2, CT2, Hp, Wp, V2 = sx
    if not (V == V2 == C16 == K16 == 16 and KT == KT2 and CT == CT2 and N2 >= N):
        return None
    if Hp < stride * (P - 1) + R or Wp < stride * (Q - 1) + S:
        return None
    rng = _loop_ranges(loops, env)
    iters = {lp.iterator for lp in loops}
    roles = [(img, N), (kt, KT), (oj, P), (oi, Q), (ofm, 16), (ct, CT), (kj, R), (ki, S), (ifm, 16)]
    used = [e.variables() & iters for e, _ in roles]
    if any(len(u & v) for i, u in enumerate(used) for v in used[i + 1:]):
        return None
    if not all(_role_ok(e, rng, ext, iters) for e, ext in roles):
        return None
    want = N * KT * P * Q * 16 * CT * R * S * 16
    if _count(list(loops), env) != want:
        return None
    par = next((lp for lp in loops if lp.parallel), None)
    role = None
    if par is not None:
        names = ["img", "kt", "oj", "oi", "ofm", "ct", "kj", "ki", "ifm"]
        role = next((nm for nm, u in zip(names, used) if par.iterator in u), None)
    return ConvPlan(nest.name, tgt.array, filt.array, inp.array, N, KT, CT, P, Q, R, S, stride,
                    Hp, Wp, parallel_role=role)


def _match_gemm(nest, stmt, loops, env, shapes):
    ops = _product_operands(stmt.expr)
    tgt = stmt.target
    if stmt.op != "+=" or ops is None or len(tgt.indices) != 2:
        return None
    a, b = ops
    i, j = tgt.indices
    if len(a.indices) != 2 or len(b.indices) != 2:
        return None
    if not (a.indices[0] == i and b.indices[1] == j and a.indices[1] == b.indices[0]):
        a, b = b, a
        if not (a.indices[0] == i and b.indices[1] == j and a.indices[1] == b.indices[0]):
            return None
    k = a.indices[1]
    M, N = shapes[tgt.array]
    Ma, K = shapes[a.array]
    Kb, Nb = shapes[b.array]
    if not (Ma >= M and Nb >= N and Kb >= K):
        return None
    rng = _loop_ranges(loops, env)
    iters = {lp.iterator for lp in loops}
    roles = [(i, M), (j, N), (k, K)]
    used = [e.variables() & iters for e, _ in roles]
    if any(len(u & v) for x, u in enumerate(used) for v in used[x + 1:]):
        return None
    # the reduction extent is the loop range, not the array extent
    kext = K
    if len(used[2]) == 1 and k == Affine.var(next(iter(used[2]))):
        kext = rng[next(iter(used[2]))][1] + 1
    roles[2] = (k, kext)
    if not all(_role_ok(e, rng, ext, iters) for e, ext in roles):
        return None
    if _count(list(loops), env) != M * N * kext:
        return None
    par = next((lp for lp in loops if lp.parallel), None)
    role = None
    if par is not None:
        role = next((nm for nm, u in zip("ijk", used) if par.iterator in u), None)
    return GemmPlan(nest.name, tgt.array, a.array, b.array, M, N, kext, parallel_role=role)


def _match_eltwise(nest, stmt, loops, env, shapes):
    """y = act(y * s + b) over the target, every part optional but one."""
    tgt = stmt.target
    if stmt.op != "=":
        return None
    e = stmt.expr
    relu6 = relu = False
    if isinstance(e, Call) and e.fn == "min" and len(e.args) == 2 and e.args[1] == Num(6.0):
        relu6, e = True, e.args[0]
    if isinstance(e, Call) and e.fn == "max" and len(e.args) == 2 and e.args[1] == Num(0.0):
        relu, e = True, e.args[0]
    elif relu6:
        return None

    def axes_of(acc):
        axes = []
        for ix in acc.indices:
            pos = [d for d, t in enumerate(tgt.indices) if t == ix]
            if len(pos) != 1:
                return None
            axes.append(pos[0])
        return tuple(axes)

    bias = scale = None
    axes = s_axes = ()
    if isinstance(e, BinOp) and e.op == "+" and isinstance(e.right, Access):
        axes = axes_of(e.right)
        if axes is None:
            return None
        bias, e = e.right.array, e.left
    if isinstance(e, BinOp) and e.op == "*" and isinstance(e.right, Access) \
            and isinstance(e.left, Access) and e.left.array == tgt.array:
        s_axes = axes_of(e.right)
        if s_axes is None:
            return None
        scale, e = e.right.array, e.left
    if not (isinstance(e, Access) and e.array == tgt.array and e.indices == tgt.indices):
        return None
    if not (relu or bias or scale):
        return None
    if tgt.array in (bias, scale):
        return None
    rng = _loop_ranges(loops, env)
    iters = {lp.iterator for lp in loops}
    ext = shapes[tgt.array]
    used = [ix.variables() & iters for ix in tgt.indices]
    if any(len(u & v) for x, u in enumerate(used) for v in used[x + 1:]):
        return None
    if not all(_role_ok(ix, rng, n, iters) for ix, n in zip(tgt.indices, ext)):
        return None
    if _count(list(loops), env) != int(np.prod(ext)):
        return None
    return EltwisePlan(nest.name, tgt.array, bias, relu, relu6, axes, scale, s_axes)


def _covers(plan, shapes) -> bool:
    """The heavy nest writes every element of its output array."""
    if isinstance(plan, ConvPlan):
        return tuple(shapes[plan.out]) == (plan.N, plan.KT, plan.P, plan.Q, 16)
    return tuple(shapes[plan.C]) == (plan.M, plan.N)


def _expand(nests) -> list:
    """FusedNest -> its operator pair in execution order (intervening nests after)."""
    out = []
    for n in nests:
        pr = getattr(n, "pair", None)
        if pr is None:
            out.append(n)
        elif pr.ew_first:
            out += [pr.eltwise, pr.heavy, *pr.between]
        else:
            out += [pr.heavy, pr.eltwise, *pr.between]
    return out


def plan_program(nests: Sequence[LoopNest], binding: Mapping[str, int]) -> list:
    """Recognise every nest; fuse an element-wise nest into the preceding heavy one
    when Alg. 3's conditions hold.  They are checked structurally on the matched
    nests (fusion.can_fuse enumerates, which only suits desk-sized bindings):
    (1) W_hy = W_ew -- the element-wise nest targets the heavy nest's output array
        and both cover all of it (the matchers prove each nest onto its array);
    (2) element-wise -- matched as one instance per element (count = |array|,
        injective subscripts), reading the target only at the element it writes;
    (3) nothing in between -- the nests are adjacent in the program."""
    nests = _expand(nests)
    plans: list = []
    shapes_all: dict = {}
    for nest in nests:
        if nest.has_kernel_call():
            if nest.microkernel is None:
                raise InterpreterError(f"cannot execute opaque kernel call in {nest.name!r}")
            nest = substitute_microkernel(nest)
        if any(isinstance(n, KernelCall) for n in walk(nest.body)):
            raise InterpreterError(f"cannot execute opaque kernel call in {nest.name!r}")
        shapes = nest.shapes(binding)
        shapes_all.update(shapes)
        env = {p: int(binding[p]) for p in nest.params}
        stmt, loops = _single_stmt(nest)
        for acc in (stmt.target,) + stmt.read_accesses():
            if acc.array not in shapes:
                raise InterpreterError(f"array {acc.array!r} has no extent")
        plan = (_match_conv(nest, stmt, loops, env, shapes)
                or _match_gemm(nest, stmt, loops, env, shapes)
                or _match_eltwise(nest, stmt, loops, env, shapes))
        if plan is None:
            raise InterpreterError(
                f"nest {nest.name!r} is not a blocked convolution, GEMM or element-wise "
                "epilogue of one; the B200 executor runs only those (no CPU fallback)")
        if isinstance(plan, EltwisePlan) and plans and not isinstance(plans[-1], EltwisePlan) \
                and plans[-1].epilogue is None:
            heavy = plans[-1]
            out = heavy.out if isinstance(heavy, ConvPlan) else heavy.C
            axes = (1, 4) if isinstance(heavy, ConvPlan) else (1,)
            if plan.target == out and plan.channel_axes_ok(axes) and _covers(heavy, shapes_all):
                heavy.epilogue = plan
                continue
        plans.append(plan)
    return plans


# ----------------------------------------------------------------------------- execution
def make_inputs(nest: LoopNest, binding: Mapping[str, int], seed: int = 0) -> dict:
    """Seeded standard-normal contents for every array (the reference's
    `make_inputs`, simcache.py:79-86): one PCG64 stream, arrays in name order."""
    rng = np.random.default_rng(seed)
    return {name: rng.standard_normal(int(np.prod(shape)) if shape else 1)
            for name, shape in sorted(nest.shapes(binding).items())}


def _as_float32_device(torch, arr, shape, device):
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(arr, dtype=np.float32)
                                              .ravel()[:int(np.prod(shape))]))
    return t.reshape(shape).to(device)


def _epilogue_args(ep, arrays, K: int) -> dict:
    """ops keyword arguments of an element-wise plan (device bias / scale vectors)."""
    if ep is None:
        return {}
    def vec(name):
        return None if name is None else arrays[name].reshape(-1)[:K].contiguous()
    return {"bias": vec(ep.bias), "scale": vec(ep.scale), "relu": ep.relu and not ep.relu6,
            "relu6": ep.relu6}


def execute(nests, binding: Mapping[str, int], inputs: Mapping[str, np.ndarray],
            mode: str = "3xtf32", device=None, keep_on_device: bool = False) -> dict:
    """Run a nest / Program on the GPU.  Returns {array: flat float64 ndarray}
    (or torch tensors with keep_on_device=True)."""
    import torch
    from . import ops

    if isinstance(nests, Program):
        nests = list(nests.nests)
    elif isinstance(nests, LoopNest):
        nests = [nests]
    nests = _expand(nests)
    missing = sorted({p for n in nests for p in n.params if p not in binding})
    if missing:
        raise UnboundParameterError(f"unbound parameters: {missing}")
    plans = plan_program(nests, binding)
    shapes = {}
    for n in nests:
        shapes.update(n.shapes(binding))
    dev = torch.device(device) if device is not None else torch.device("cuda")
    arrays: dict = {}
    nonzero: dict = {}   # host-side: does the incoming array hold anything but zeros?
    for name, shape in shapes.items():
        if name not in inputs:
            raise InterpreterError(f"input array {name!r} missing")
        need = int(np.prod(shape)) if shape else 1
        host = inputs[name]
        if isinstance(host, np.ndarray) or not hasattr(host, "is_cuda"):
            host = np.asarray(host)
            if host.size < need:
                raise InterpreterError(f"input array {name!r} too small")
            nonzero[name] = bool(np.any(host.ravel()[:need] != 0))
            arrays[name] = _as_float32_device(torch, host, shape, dev)
        else:                          # a device tensor (keep_on_device chaining)
            if host.numel() < need:
                raise InterpreterError(f"input array {name!r} too small")
            nonzero[name] = True       # unknown without a device sync: accumulate
            arrays[name] = host.reshape(-1)[:need].to(dev, torch.float32).reshape(shape)
    for plan in plans:
        if isinstance(plan, ConvPlan):
            y0 = arrays[plan.out]
            x = arrays[plan.inp][:plan.N]
            w = arrays[plan.filt]
            ep = plan.epilogue
            kw = _epilogue_args(ep, arrays, plan.KT * 16)
            accumulate = nonzero.get(plan.out, True)
            fuse = ep is not None and not accumulate
            y = ops.conv2d_nchw16c(x.contiguous(), w.contiguous(), stride=plan.stride, pad=0,
                                   mode=mode, **(kw if fuse else {}))
            y = y[:, :, :plan.P, :plan.Q, :].contiguous()
            if accumulate:           # `+=` onto non-zero incoming contents (+ the epilogue)
                ops.accumulate_(y, y0.contiguous(), **kw)
            arrays[plan.out] = y
            nonzero[plan.out] = True
        elif isinstance(plan, GemmPlan):
            a = arrays[plan.A][:plan.M, :plan.K].contiguous()
            b = arrays[plan.B][:plan.K, :plan.N].contiguous()
            ep = plan.epilogue
            # `+=` onto non-zero incoming C: beta = 1 inside the kernel, C updated in place
            beta = 1.0 if nonzero.get(plan.C, True) else 0.0
            c = arrays[plan.C].contiguous()
            ekw = {}
            if ep is not None:
                vec = lambda nm: None if nm is None else arrays[nm].reshape(-1)[:plan.N].contiguous()  # noqa: E731
                ekw = {"bias": vec(ep.bias), "scale": vec(ep.scale), "relu": ep.relu and not ep.relu6,
                       "relu6": ep.relu6}
            ops.gemm(a, b, c, beta=beta, mode=mode, **ekw)
            arrays[plan.C] = c
            nonzero[plan.C] = True
        else:  # stand-alone element-wise nest (no preceding heavy nest to fuse into)
            y = arrays[plan.target]
            if y.dim() == 5 and y.shape[-1] == 16 and plan.channel_axes_ok((1, 4)):
                y = y.contiguous()
                ops.bias_relu_(y, **_epilogue_args(plan, arrays, y.shape[1] * 16))
                arrays[plan.target] = y
                nonzero[plan.target] = True
                continue
            raise InterpreterError(f"element-wise nest {plan.nest!r} is only supported on nChw16c "
                                   "conv outputs (channel-indexed bias / scale) or fused after a "
                                   "GEMM")
    if keep_on_device:
        return arrays
    return {k: v.detach().to("cpu", torch.float64).reshape(-1).numpy() for k, v in arrays.items()}


def interpret(nest, binding: Mapping[str, int], seed: int = 0,
              inputs: Mapping[str, np.ndarray] | None = None, collect_trace: bool = True,
              mode: str = "3xtf32"):
    """Drop-in for `looprank.simcache.interpret` (simcache.py:89-204), same
    signature and defaults: returns (arrays, trace).  The arrays are computed on
    the B200.  The trace (collect_trace=True, the reference's default) is a
    `trace.LazyTrace`: the reference's TraceRecord sequence, generated on the host
    from the nest structure when first used (it does not depend on the values);
    for a Program, a tuple with one LazyTrace per nest.  collect_trace=False
    returns None, as the reference returns an empty Trace's records."""
    from .trace import LazyTrace
    first = nest.nests[0] if isinstance(nest, Program) else nest
    if inputs is None:
        inputs = make_inputs(first, binding, seed)
    arrays = execute(nest, binding, inputs, mode=mode)
    if not collect_trace:
        return arrays, None
    if isinstance(nest, Program):
        return arrays, tuple(LazyTrace(n, binding) for n in nest.nests)
    return arrays, LazyTrace(nest, binding)
