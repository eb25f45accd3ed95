"""Loop-nest language (`.pdl`) front end: scanner, parser, affine algebra and IR.

Host-side mirror of the reference's `looprank.loopdsl` entry points
(/root/reference/pkg/src/looprank/loopdsl.py): the same source language and
the same IR vocabulary (`Loop`, `Access`, `Statement`, `LoopNode`, `StmtNode`,
`KernelCall`, `KernelRegion`, `MicrokernelSpec`, `LoopNest`, `Program`), the
same entry points (`parse` loopdsl.py:732-739, `parse_program` :728-729,
`substitute_microkernel` :747-760, `reinstate_microkernel` :763-784,
`pretty` :944-983, `to_json` :999-1032) and the same error classes
(`ParseError` with line:col, `NonAffineError`, loopdsl.py:36-48).

Language summary (identical surface syntax):

    param M, N, K;
    array C[M][N];
    gemm: parallel for (i = 0; i < M; i++) {
      for (j = 0; j < N; j += 1) {
        for (k = 0; k < min(K, 64); k++) {
          S: C[i][j] += A[i][k] * B[k][j];
    } } }

* `parallel` or `#pragma omp parallel for` marks a loop parallel (the batch
  sharding axis of the executor);
* `#pragma microkernel NAME(ARGS) { band }` declares the loop band an opaque
  tuned routine replaces -- on B200 that routine is the tcgen05 tile engine;
* `x = <affine>;` inside a loop declares a derived iterator, folded into the
  subscripts at parse time;
* bounds / subscripts must be affine; values may use + - * /, min, max,
  numeric literals and array references (no named scalars).

This module is pure Python (no torch / CUDA) so the IR tooling runs anywhere.
"""
from __future__ import annotations

import json
import re
from dataclasses import dataclass, field, replace
from typing import Iterable, Iterator, Mapping, Sequence

__all__ = [
    "Affine", "Loop", "Access", "Num", "Neg", "BinOp", "Call", "Statement", "LoopNode",
    "StmtNode", "KernelCall", "KernelRegion", "MicrokernelSpec", "LoopNest", "Program",
    "LoopDslError", "ParseError", "NonAffineError", "UnboundParameterError", "parse",
    "parse_program", "substitute_microkernel", "reinstate_microkernel", "pretty",
    "pretty_program", "to_json", "dump_json", "walk", "statements_with_loops",
]


class LoopDslError(Exception):
    """Malformed or unsupported loop nest."""


class ParseError(LoopDslError):
    """Syntax error, reported as ``line:col: message`` when a position is known."""

    def __init__(self, message: str, line: int = 0, col: int = 0):
        self.line, self.col = line, col
        super().__init__(f"{line}:{col}: {message}" if line else message)


class NonAffineError(ParseError):
    """A bound or subscript that is not affine in iterators and parameters."""


class UnboundParameterError(LoopDslError):
    """A size parameter has no value in the binding."""


# ----------------------------------------------------------------------------- affine
class Affine:
    """Integer affine form  sum_i c_i * v_i + c0  (immutable, hashable)."""

    __slots__ = ("terms", "c0")

    def __init__(self, terms: Mapping[str, int] | None = None, c0: int = 0):
        t = {}
        for name, c in (terms or {}).items():
            if int(c) != c:
                raise TypeError("affine coefficients are integers")
            if c:
                t[name] = int(c)
        object.__setattr__(self, "terms", dict(sorted(t.items())))
        object.__setattr__(self, "c0", int(c0))

    def __setattr__(self, *_):
        raise AttributeError("Affine is immutable")

    # construction ------------------------------------------------------------
    @staticmethod
    def const(v: int) -> "Affine":
        return Affine(None, v)

    @staticmethod
    def var(name: str) -> "Affine":
        return Affine({name: 1})

    @staticmethod
    def lift(x) -> "Affine":
        if isinstance(x, Affine):
            return x
        if isinstance(x, str):
            return Affine.var(x)
        return Affine.const(int(x))

    # algebra -----------------------------------------------------------------
    def __add__(self, other):
        o = Affine.lift(other)
        t = dict(self.terms)
        for k, v in o.terms.items():
            t[k] = t.get(k, 0) + v
        return Affine(t, self.c0 + o.c0)

    __radd__ = __add__

    def __neg__(self):
        return Affine({k: -v for k, v in self.terms.items()}, -self.c0)

    def __sub__(self, other):
        return self + (-Affine.lift(other))

    def __rsub__(self, other):
        return Affine.lift(other) - self

    def scale(self, k: int) -> "Affine":
        return Affine({n: c * k for n, c in self.terms.items()}, self.c0 * k)

    def __mul__(self, other):
        o = Affine.lift(other)
        if o.is_const():
            return self.scale(o.c0)
        if self.is_const():
            return o.scale(self.c0)
        raise NonAffineError("product of two non-constant affine expressions")

    __rmul__ = __mul__

    def is_const(self) -> bool:
        return not self.terms

    def coeff(self, name: str) -> int:
        return self.terms.get(name, 0)

    def variables(self) -> frozenset[str]:
        return frozenset(self.terms)

    def subst(self, env: Mapping[str, "Affine | int"]) -> "Affine":
        out = Affine.const(self.c0)
        for n, c in self.terms.items():
            out = out + (Affine.lift(env[n]).scale(c) if n in env else Affine({n: c}))
        return out

    def eval(self, env: Mapping[str, int]) -> int:
        total = self.c0
        for n, c in self.terms.items():
            if n not in env:
                raise UnboundParameterError(f"no value for {n!r}")
            total += c * int(env[n])
        return total

    def __eq__(self, other):
        if not isinstance(other, Affine):
            try:
                other = Affine.lift(other)
            except (TypeError, ValueError):
                return NotImplemented
        return self.terms == other.terms and self.c0 == other.c0

    def __hash__(self):
        return hash((tuple(self.terms.items()), self.c0))

    def text(self) -> str:
        parts = []
        for n, c in self.terms.items():
            mag = abs(c)
            body = n if mag == 1 else f"{mag}*{n}"
            parts.append(("- " if c < 0 else "+ ") + body)
        if self.c0 or not parts:
            parts.append(("- " if self.c0 < 0 else "+ ") + str(abs(self.c0)))
        s = " ".join(parts)
        return s[2:] if s.startswith("+ ") else "-" + s[2:]

    def __repr__(self):
        return f"Affine({self.text()})"


# ----------------------------------------------------------------------------- IR
@dataclass(frozen=True)
class Loop:
    iterator: str
    lower: Affine
    upper: tuple            # tuple[Affine, ...]: run while iterator < min(upper)
    step: int = 1
    parallel: bool = False

    def trip_count(self, env: Mapping[str, int]) -> int:
        lo = self.lower.eval(env)
        hi = min(u.eval(env) for u in self.upper)
        return max(0, -(-(hi - lo) // self.step))


@dataclass(frozen=True)
class Access:
    array: str
    indices: tuple          # tuple[Affine, ...]
    kind: str = "read"      # "read" | "write"


@dataclass(frozen=True)
class Num:
    value: float


@dataclass(frozen=True)
class Neg:
    operand: object


@dataclass(frozen=True)
class BinOp:
    op: str                 # + - * /
    left: object
    right: object


@dataclass(frozen=True)
class Call:
    fn: str                 # "min" | "max"
    args: tuple


@dataclass(frozen=True)
class Statement:
    label: str
    target: Access
    op: str                 # "=" | "+="
    expr: object

    def read_accesses(self) -> tuple:
        reads = list(expr_accesses(self.expr))
        if self.op == "+=":
            reads.append(replace(self.target, kind="read"))
        return tuple(reads)


@dataclass(frozen=True)
class LoopNode:
    loop: Loop
    body: tuple


@dataclass(frozen=True)
class StmtNode:
    stmt: Statement


@dataclass(frozen=True)
class KernelCall:
    name: str
    args: tuple


@dataclass(frozen=True)
class KernelRegion:
    name: str
    args: tuple
    body: tuple


@dataclass(frozen=True)
class MicrokernelSpec:
    name: str
    args: tuple
    body: tuple


@dataclass(frozen=True)
class LoopNest:
    name: str
    params: tuple
    arrays: tuple           # ((name, (Affine extents...)), ...)
    body: tuple
    microkernel: MicrokernelSpec | None = None

    def array_extents(self) -> dict:
        return dict(self.arrays)

    def loops(self) -> list:
        return [n.loop for n in walk(self.body) if isinstance(n, LoopNode)]

    def statements(self) -> list:
        return [n.stmt for n in walk(self.body) if isinstance(n, StmtNode)]

    def has_kernel_call(self) -> bool:
        return any(isinstance(n, KernelCall) for n in walk(self.body))

    def has_kernel_region(self) -> bool:
        return any(isinstance(n, KernelRegion) for n in walk(self.body))

    def shapes(self, binding: Mapping[str, int]) -> dict:
        missing = [p for p in self.params if p not in binding]
        if missing:
            raise UnboundParameterError(f"unbound parameters: {missing}")
        return {a: tuple(max(0, d.eval(binding)) for d in dims) for a, dims in self.arrays}


@dataclass(frozen=True)
class Program:
    params: tuple
    arrays: tuple
    nests: tuple


def expr_accesses(e) -> Iterator[Access]:
    if isinstance(e, Access):
        yield e
    elif isinstance(e, Neg):
        yield from expr_accesses(e.operand)
    elif isinstance(e, BinOp):
        yield from expr_accesses(e.left)
        yield from expr_accesses(e.right)
    elif isinstance(e, Call):
        for a in e.args:
            yield from expr_accesses(a)


def walk(nodes) -> Iterator:
    """Preorder over loop / region / statement nodes."""
    stack = list(reversed(tuple(nodes)))
    while stack:
        n = stack.pop()
        yield n
        if isinstance(n, (LoopNode, KernelRegion)):
            stack.extend(reversed(n.body))


def statements_with_loops(nodes, enclosing=()) -> Iterator[tuple]:
    """(statement, enclosing loops outermost-first) for every statement."""
    for n in nodes:
        if isinstance(n, LoopNode):
            yield from statements_with_loops(n.body, enclosing + (n.loop,))
        elif isinstance(n, KernelRegion):
            yield from statements_with_loops(n.body, enclosing)
        elif isinstance(n, StmtNode):
            yield n.stmt, enclosing


def rebuild(nodes, fn) -> tuple:
    out = []
    for n in nodes:
        if isinstance(n, LoopNode):
            n = LoopNode(n.loop, rebuild(n.body, fn))
        elif isinstance(n, KernelRegion):
            n = KernelRegion(n.name, n.args, rebuild(n.body, fn))
        r = fn(n)
        if r is None:
            continue
        out.extend(r if isinstance(r, (list, tuple)) else [r])
    return tuple(out)


# ----------------------------------------------------------------------------- scanner
_KEYWORDS = frozenset({"for", "param", "array", "parallel", "min", "max"})
_PUNCT2 = ("++", "+=", "<=", ">=", "==")
_PUNCT1 = set("-+*/%(){}[];:,=<>")
_OMP = re.compile(r"#pragma\s+omp\s+parallel\s+for\b")
_MK = re.compile(r"#pragma\s+microkernel\s+([A-Za-z_]\w*)\s*\(([^)]*)\)\s*$")


@dataclass
class Token:
    kind: str       # name | int | float | punct text | omp | mk | eof
    text: str
    line: int
    col: int
    extra: object = None


def scan(src: str) -> list:
    toks: list = []
    i, line, bol, n = 0, 1, 0, len(src)
    while i < n:
        ch = src[i]
        col = i - bol + 1
        if ch == "\n":
            line += 1
            i += 1
            bol = i
            continue
        if ch.isspace():
            i += 1
            continue
        if src.startswith("//", i):
            while i < n and src[i] != "\n":
                i += 1
            continue
        if ch == "#":
            j = src.find("\n", i)
            j = n if j < 0 else j
            text = src[i:j].rstrip()
            if _OMP.match(text):
                toks.append(Token("omp", text, line, col))
            else:
                m = _MK.match(text)
                if not m:
                    raise ParseError(f"malformed pragma: {text!r}", line, col)
                args = tuple(a.strip() for a in m.group(2).split(",") if a.strip())
                toks.append(Token("mk", text, line, col, (m.group(1), args)))
            i = j
            continue
        if ch.isdigit():
            j = i
            while j < n and src[j].isdigit():
                j += 1
            if j + 1 < n and src[j] == "." and src[j + 1].isdigit():
                j += 1
                while j < n and src[j].isdigit():
                    j += 1
                toks.append(Token("float", src[i:j], line, col))
            else:
                toks.append(Token("int", src[i:j], line, col))
            i = j
            continue
        if ch.isalpha() or ch == "_":
            j = i
            while j < n and (src[j].isalnum() or src[j] == "_"):
                j += 1
            toks.append(Token("name", src[i:j], line, col))
            i = j
            continue
        two = src[i:i + 2]
        if two in _PUNCT2:
            toks.append(Token(two, two, line, col))
            i += 2
            continue
        if ch in _PUNCT1:
            toks.append(Token(ch, ch, line, col))
            i += 1
            continue
        raise ParseError(f"unexpected character {ch!r}", line, col)
    toks.append(Token("eof", "", line, i - bol + 1))
    return toks


# ----------------------------------------------------------------------------- parser
class _Env:
    """Lexical environment: params, loop iterators and folded derived iterators."""

    def __init__(self, params):
        self.params = set(params)
        self.frames: list = [{}]

    def find(self, name):
        for fr in reversed(self.frames):
            if name in fr:
                return fr[name]
        return Affine.var(name) if name in self.params else None

    def bind(self, name, value, tok):
        if self.find(name) is not None:
            raise ParseError(f"identifier {name!r} shadows an existing one", tok.line, tok.col)
        self.frames[-1][name] = value


class _Reader:
    def __init__(self, src: str):
        self.toks = scan(src)
        self.pos = 0

    # token helpers -------------------------------------------------------------
    def la(self, k=0) -> Token:
        return self.toks[min(self.pos + k, len(self.toks) - 1)]

    def take(self) -> Token:
        t = self.toks[self.pos]
        if t.kind != "eof":
            self.pos += 1
        return t

    def want(self, kind: str) -> Token:
        t = self.take()
        if t.kind != kind:
            raise ParseError(f"expected {kind!r}, found {t.text!r}", t.line, t.col)
        return t

    def ident(self) -> Token:
        t = self.want("name")
        if t.text in _KEYWORDS:
            raise ParseError(f"keyword {t.text!r} used as identifier", t.line, t.col)
        return t

    def is_word(self, word, k=0) -> bool:
        t = self.la(k)
        return t.kind == "name" and t.text == word

    # program --------------------------------------------------------------------
    def program(self) -> Program:
        params: list = []
        declared: dict = {}
        raw_nests: list = []
        top = _Env(())
        while self.la().kind != "eof":
            if self.is_word("param"):
                self.take()
                params.append(self.ident().text)
                while self.la().kind == ",":
                    self.take()
                    params.append(self.ident().text)
                self.want(";")
                top.params = set(params)
            elif self.is_word("array"):
                self.take()
                name = self.ident().text
                dims = []
                while self.la().kind == "[":
                    self.take()
                    dims.append(self.affine(top))
                    self.want("]")
                self.want(";")
                declared[name] = tuple(dims)
            else:
                raw_nests.append(self.nest(params, declared, f"op{len(raw_nests)}"))
        if not raw_nests:
            t = self.la()
            raise ParseError("statement required: no loop nest found", t.line, t.col)
        nests = [replace(n, arrays=tuple(_infer_extents(n, declared).items())) for n in raw_nests]
        merged = _merge_extents(nests)
        nests = [replace(n, arrays=merged) for n in nests]
        return Program(tuple(params), merged, tuple(nests))

    def nest(self, params, declared, default) -> LoopNest:
        name = default
        if self.la().kind == "name" and self.la().text not in _KEYWORDS and self.la(1).kind == ":":
            name = self.take().text
            self.take()
        env = _Env(params)
        mk: list = []
        node = self.loop_or_none(env, mk)
        if node is None:
            t = self.la()
            raise ParseError("expected a loop", t.line, t.col)
        return LoopNest(name, tuple(params), tuple(declared.items()), (node,), mk[0] if mk else None)

    def loop_or_none(self, env, mk):
        par = False
        if self.la().kind == "omp" or self.is_word("parallel"):
            self.take()
            par = True
        if not self.is_word("for"):
            if par:
                t = self.la()
                raise ParseError("expected 'for' after parallel marker", t.line, t.col)
            return None
        self.take()
        self.want("(")
        it = self.ident()
        self.want("=")
        lower = self.affine(env)
        self.want(";")
        c = self.ident()
        if c.text != it.text:
            raise ParseError(f"loop condition must test {it.text!r}", c.line, c.col)
        self.want("<")
        if self.is_word("min"):
            self.take()
            self.want("(")
            ups = [self.affine(env)]
            while self.la().kind == ",":
                self.take()
                ups.append(self.affine(env))
            self.want(")")
        else:
            ups = [self.affine(env)]
        self.want(";")
        u = self.ident()
        if u.text != it.text:
            raise ParseError(f"loop increment must update {it.text!r}", u.line, u.col)
        t = self.take()
        if t.kind == "++":
            step = 1
        elif t.kind == "+=":
            st = self.want("int")
            step = int(st.text)
            if step < 1:
                raise ParseError("loop step must be positive", st.line, st.col)
        else:
            raise ParseError("expected '++' or '+= <int>'", t.line, t.col)
        self.want(")")
        env.frames.append({})
        env.bind(it.text, Affine.var(it.text), it)
        body = self.body(env, mk)
        env.frames.pop()
        if not body:
            raise ParseError("statement required: empty loop body", it.line, it.col)
        return LoopNode(Loop(it.text, lower, tuple(ups), step, par), body)

    def body(self, env, mk) -> tuple:
        if self.la().kind != "{":
            return tuple(self.item(env, mk))
        self.take()
        items: list = []
        while self.la().kind != "}":
            if self.la().kind == "eof":
                t = self.la()
                raise ParseError("unterminated block", t.line, t.col)
            items.extend(self.item(env, mk))
        self.take()
        return tuple(items)

    def item(self, env, mk) -> list:
        t = self.la()
        if t.kind == "mk":
            self.take()
            if mk:
                raise ParseError("at most one microkernel region per nest", t.line, t.col)
            env.frames.append({})
            band = self.body(env, mk)
            env.frames.pop()
            if not band or not all(isinstance(n, LoopNode) for n in band):
                raise ParseError("microkernel body must be a loop band", t.line, t.col)
            name, args = t.extra
            mk.append(MicrokernelSpec(name, args, band))
            return [KernelCall(name, args)]
        loop = self.loop_or_none(env, mk)
        if loop is not None:
            return [loop]
        if t.kind != "name":
            raise ParseError(f"expected statement, found {t.text!r}", t.line, t.col)
        label = ""
        if self.la(1).kind == ":":
            label = self.take().text
            self.take()
        if not label and self.la(1).kind == "=":
            nm = self.take()
            self.take()
            val = self.affine(env)
            self.want(";")
            env.bind(nm.text, val, nm)
            return []
        return [StmtNode(self.statement(env, label))]

    def statement(self, env, label) -> Statement:
        arr = self.ident()
        idx = self.subscripts(env)
        if not idx:
            raise ParseError(f"expected subscripts on {arr.text!r}", arr.line, arr.col)
        t = self.take()
        if t.kind not in ("=", "+="):
            raise ParseError("expected '=' or '+='", t.line, t.col)
        expr = self.vexpr(env)
        self.want(";")
        return Statement(label, Access(arr.text, idx, "write"), t.kind, expr)

    def subscripts(self, env) -> tuple:
        out = []
        while self.la().kind == "[":
            self.take()
            out.append(self.affine(env))
            self.want("]")
        return tuple(out)

    # affine expressions -------------------------------------------------------
    def affine(self, env) -> Affine:
        acc = self.aterm(env)
        while self.la().kind in ("+", "-"):
            op = self.take().kind
            rhs = self.aterm(env)
            acc = acc + rhs if op == "+" else acc - rhs
        return acc

    def aterm(self, env) -> Affine:
        acc = self.afactor(env)
        while self.la().kind == "*":
            star = self.take()
            rhs = self.afactor(env)
            if not (acc.is_const() or rhs.is_const()):
                raise NonAffineError("non-affine index: product of two non-constant expressions",
                                     star.line, star.col)
            acc = acc * rhs
        return acc

    def afactor(self, env) -> Affine:
        t = self.take()
        if t.kind == "-":
            return -self.afactor(env)
        if t.kind == "+":
            return self.afactor(env)
        if t.kind == "int":
            return Affine.const(int(t.text))
        if t.kind == "(":
            inner = self.affine(env)
            self.want(")")
            return inner
        if t.kind == "name":
            if t.text in _KEYWORDS:
                raise ParseError(f"keyword {t.text!r} in expression", t.line, t.col)
            v = env.find(t.text)
            if v is None:
                raise ParseError(f"undeclared identifier {t.text!r}", t.line, t.col)
            return v
        raise ParseError(f"expected affine expression, found {t.text!r}", t.line, t.col)

    # value expressions --------------------------------------------------------
    def vexpr(self, env):
        acc = self.vterm(env)
        while self.la().kind in ("+", "-"):
            op = self.take().kind
            acc = BinOp(op, acc, self.vterm(env))
        return acc

    def vterm(self, env):
        acc = self.vfactor(env)
        while self.la().kind in ("*", "/"):
            op = self.take().kind
            acc = BinOp(op, acc, self.vfactor(env))
        return acc

    def vfactor(self, env):
        t = self.take()
        if t.kind == "-":
            inner = self.vfactor(env)
            return Num(-inner.value) if isinstance(inner, Num) else Neg(inner)
        if t.kind in ("int", "float"):
            return Num(float(t.text))
        if t.kind == "(":
            inner = self.vexpr(env)
            self.want(")")
            return inner
        if t.kind == "name" and t.text in ("min", "max"):
            self.want("(")
            args = [self.vexpr(env)]
            while self.la().kind == ",":
                self.take()
                args.append(self.vexpr(env))
            self.want(")")
            return Call(t.text, tuple(args))
        if t.kind == "name":
            if t.text in _KEYWORDS:
                raise ParseError(f"keyword {t.text!r} in expression", t.line, t.col)
            if self.la().kind != "[":
                raise ParseError(f"scalar operand {t.text!r}: only array references and "
                                 "numeric literals are allowed", t.line, t.col)
            return Access(t.text, self.subscripts(env), "read")
        raise ParseError(f"expected expression, found {t.text!r}", t.line, t.col)


def _bounds(expr: Affine, ranges: Mapping[str, tuple], upper: bool) -> Affine:
    """Interval bound of an affine expression given iterator ranges (params stay)."""
    out = Affine.const(expr.c0)
    for n, c in expr.terms.items():
        if n in ranges:
            lo, hi = ranges[n]
            out = out + (hi if (c > 0) == upper else lo).scale(c)
        else:
            out = out + Affine({n: c})
    return out


def _infer_extents(nest: LoopNest, declared: Mapping[str, tuple]) -> dict:
    """Check declared ranks; infer extents of undeclared arrays (max index + 1)."""
    found: dict = {}
    body = nest.body
    if nest.microkernel is not None:
        spec = nest.microkernel
        body = rebuild(body, lambda n: KernelRegion(n.name, n.args, spec.body)
                       if isinstance(n, KernelCall) else n)

    def visit(nodes, ranges):
        for n in nodes:
            if isinstance(n, LoopNode):
                lp = n.loop
                lo = _bounds(lp.lower, ranges, upper=False)
                hi = _bounds(lp.upper[0] - 1, ranges, upper=True)
                visit(n.body, {**ranges, lp.iterator: (lo, hi)})
            elif isinstance(n, KernelRegion):
                visit(n.body, ranges)
            elif isinstance(n, StmtNode):
                st = n.stmt
                for acc in (st.target,) + st.read_accesses():
                    if acc.array in declared and len(declared[acc.array]) != len(acc.indices):
                        raise ParseError(f"array {acc.array!r} has rank "
                                         f"{len(declared[acc.array])}, subscripted with "
                                         f"{len(acc.indices)} indices")
                    ext = found.setdefault(acc.array, [Affine.const(0)] * len(acc.indices))
                    for d, ix in enumerate(acc.indices):
                        ext[d] = _affine_max(ext[d], _bounds(ix, ranges, upper=True) + 1)

    visit(body, {})
    out = dict(declared)
    for name, dims in found.items():
        out.setdefault(name, tuple(dims))
    return out


def _affine_max(a: Affine, b: Affine) -> Affine:
    d = a - b
    if d.is_const():
        return a if d.c0 >= 0 else b
    return a + b  # sound over-approximation (extents only size buffers)


def _merge_extents(nests) -> tuple:
    merged: dict = {}
    for n in nests:
        for name, dims in n.arrays:
            if name not in merged:
                merged[name] = dims
                continue
            if len(merged[name]) != len(dims):
                raise ParseError(f"array {name!r} used with inconsistent rank")
            merged[name] = tuple(_affine_max(a, b) for a, b in zip(merged[name], dims))
    return tuple(merged.items())


def parse_program(text: str) -> Program:
    """All nests of a `.pdl` source (one shared array namespace)."""
    return _Reader(text).program()


def parse(text: str, name: str | None = None) -> LoopNest:
    """A `.pdl` source holding exactly one nest."""
    prog = parse_program(text)
    if len(prog.nests) != 1:
        raise ParseError(f"expected one loop nest, found {len(prog.nests)}")
    nest = prog.nests[0]
    if name is not None and re.fullmatch(r"op\d+", nest.name):
        nest = replace(nest, name=name)
    return nest


# ----------------------------------------------------------------------------- microkernel
def substitute_microkernel(nest: LoopNest) -> LoopNest:
    """Inline the pragma's loop band in place of the opaque call (marked region)."""
    spec = nest.microkernel
    if spec is None or not nest.has_kernel_call():
        return nest
    return replace(nest, body=rebuild(nest.body, lambda n: KernelRegion(spec.name, spec.args, spec.body)
                                      if isinstance(n, KernelCall) and n.name == spec.name else n))


def reinstate_microkernel(nest: LoopNest) -> LoopNest:
    """Put the opaque call back; refuses if the marked band was modified."""
    spec = nest.microkernel
    if spec is None:
        raise LoopDslError(f"nest {nest.name!r} has no microkernel spec")
    regions = [n for n in walk(nest.body) if isinstance(n, KernelRegion)]
    if not regions:
        raise LoopDslError(f"nest {nest.name!r} has no marked band to reinstate")
    if any(r.body != spec.body for r in regions):
        raise LoopDslError("microkernel band was modified; refusing to reinstate")
    return replace(nest, body=rebuild(nest.body, lambda n: KernelCall(spec.name, spec.args)
                                      if isinstance(n, KernelRegion) and n.name == spec.name else n))


# ----------------------------------------------------------------------------- printing
def render_expr(e, prec: int = 0) -> str:
    if isinstance(e, Num):
        v = e.value
        return str(int(v)) if v == int(v) and abs(v) < 1e15 else repr(v)
    if isinstance(e, Neg):
        return "-" + render_expr(e.operand, 3)
    if isinstance(e, Access):
        return e.array + "".join(f"[{ix.text()}]" for ix in e.indices)
    if isinstance(e, Call):
        return f"{e.fn}({', '.join(render_expr(a) for a in e.args)})"
    if isinstance(e, BinOp):
        mine = 1 if e.op in "+-" else 2
        s = f"{render_expr(e.left, mine)} {e.op} {render_expr(e.right, mine + 1)}"
        return f"({s})" if mine < prec else s
    raise TypeError(f"unknown expression node {e!r}")


def pretty(nest: LoopNest) -> str:
    lines: list = []
    if nest.params:
        lines.append("param " + ", ".join(nest.params) + ";")
    for a, dims in nest.arrays:
        lines.append(f"array {a}" + "".join(f"[{d.text()}]" for d in dims) + ";")
    if lines:
        lines.append("")

    def emit(nodes, depth):
        ind = "  " * depth
        for n in nodes:
            if isinstance(n, LoopNode):
                lp = n.loop
                up = lp.upper[0].text() if len(lp.upper) == 1 else \
                    "min(" + ", ".join(u.text() for u in lp.upper) + ")"
                inc = f"{lp.iterator}++" if lp.step == 1 else f"{lp.iterator} += {lp.step}"
                pre = "parallel " if lp.parallel else ""
                lines.append(f"{ind}{pre}for ({lp.iterator} = {lp.lower.text()}; "
                             f"{lp.iterator} < {up}; {inc}) {{")
                emit(n.body, depth + 1)
                lines.append(ind + "}")
            elif isinstance(n, (KernelCall, KernelRegion)):
                lines.append(f"{ind}#pragma microkernel {n.name}({', '.join(n.args)})")
                band = n.body if isinstance(n, KernelRegion) else \
                    (nest.microkernel.body if nest.microkernel else ())
                lines.append(ind + "{")
                emit(band, depth + 1)
                lines.append(ind + "}")
            elif isinstance(n, StmtNode):
                s = n.stmt
                lab = f"{s.label}: " if s.label else ""
                lines.append(f"{ind}{lab}{render_expr(s.target)} {s.op} {render_expr(s.expr)};")

    first = len(lines)
    emit(nest.body, 0)
    lines[first] = f"{nest.name}: {lines[first]}"
    return "\n".join(lines) + "\n"


def pretty_program(prog: Program) -> str:
    head = ["param " + ", ".join(prog.params) + ";"] if prog.params else []
    head += [f"array {a}" + "".join(f"[{d.text()}]" for d in dims) + ";" for a, dims in prog.arrays]
    chunks = ["\n".join(head) + "\n"] if head else []
    chunks += [pretty(replace(n, params=(), arrays=())) for n in prog.nests]
    return "\n".join(chunks)


def to_json(nest: LoopNest) -> dict:
    def node(n):
        if isinstance(n, LoopNode):
            lp = n.loop
            return {"kind": "loop", "iterator": lp.iterator, "lower": lp.lower.text(),
                    "upper": [u.text() for u in lp.upper], "step": lp.step,
                    "parallel": lp.parallel, "body": [node(c) for c in n.body]}
        if isinstance(n, KernelRegion):
            return {"kind": "kernel_region", "name": n.name, "args": list(n.args),
                    "body": [node(c) for c in n.body]}
        if isinstance(n, KernelCall):
            return {"kind": "kernel_call", "name": n.name, "args": list(n.args)}
        s = n.stmt
        return {"kind": "statement", "label": s.label, "op": s.op, "expr": render_expr(s.expr),
                "accesses": [{"array": a.array, "kind": a.kind,
                              "indices": [i.text() for i in a.indices]}
                             for a in (s.target,) + s.read_accesses()]}

    mk = nest.microkernel
    return {"version": 1, "name": nest.name, "params": list(nest.params),
            "arrays": {a: [d.text() for d in dims] for a, dims in nest.arrays},
            "loops": [{"iterator": l.iterator, "step": l.step, "parallel": l.parallel}
                      for l in nest.loops()],
            "statements": [{"label": s.label or f"S{i}"} for i, s in enumerate(nest.statements())],
            "body": [node(n) for n in nest.body],
            "microkernel": None if mk is None else {"name": mk.name, "args": list(mk.args),
                                                   "body": [node(n) for n in mk.body]}}


def dump_json(nest: LoopNest) -> str:
    return json.dumps(to_json(nest), indent=2, sort_keys=True)
