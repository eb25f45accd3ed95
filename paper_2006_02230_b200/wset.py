"""Working sets (PolyDL Alg. 1) -- exact enumeration form and the B200 tile
engine's closed form.

1. `working_sets(nest, binding)` mirrors `looprank.wset.working_sets`
   (/root/reference/pkg/src/looprank/wset.py:166-207) with the reference's
   definitions (depend.py:1-125):
     * a dependence exists for every ordered pair of references to one array
       (RAR / RAW / WAR / WAW) that touch the same element at a strictly later
       schedule point;
     * if source and target can differ in a shared parallel iterator the entry
       is WS_par: the footprint of all iterations with the iterators outside the
       parallel loop fixed at their lexicographic minimum (wset.py:113-163);
     * otherwise, from the lexicographically first source iteration, WS_min /
       WS_max are the footprints (distinct elements, summed over arrays) of all
       accesses scheduled between the source and its first / last target,
       inclusive (wset.py:178-195).
   The reference evaluates these with a polyhedral set engine; here the nest is
   simply enumerated in schedule order, which is exact and fast for the
   desk-size bindings Alg. 1 is validated on (the reference needs 100-2000 s
   per tiny tiled nest; this takes milliseconds).  Tests pin it
   to the paper's worked example (WS_min = 2K+3, WS_max = NK+N+1)
   and to the reference itself at small bindings.

2. `tile_working_sets(layer, variant)` is the closed form for the schedules the
   B200 ranker chooses between: the tile engine's explicit buffers (SMEM
   stages, TMEM accumulators and A slots) and the L2-resident reuse (the weight
   slice of an N-tile shared by all M-tiles; the input halo shared between
   neighbouring tiles), plus the compulsory HBM stream.  These feed Alg. 2
   (`machine.assign_to_caches`) and Eq. 1 (`rank.cost`) exactly as the CPU
   working sets did.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

from .loopnest import (Access, KernelRegion, LoopNest, LoopNode, StmtNode, UnboundParameterError,
                       substitute_microkernel)


class WorkingSetError(Exception):
    pass


@dataclass(frozen=True)
class WorkingSetEntry:
    dep_id: str
    kind: str        # RAR / RAW / WAR / WAW  (or "buffer" / "reuse" / "stream" for tiles)
    array: str
    variant: str     # "par" | "min" | "max" | level hint
    elements: int

    def key(self) -> str:
        return f"{self.dep_id}:{self.variant}"

    def size_bytes(self, dtype_size: int = 4) -> int:
        return self.elements * dtype_size


@dataclass(frozen=True)
class WorkingSetReport:
    nest: str
    binding: tuple
    entries: tuple

    def binding_dict(self) -> dict:
        return dict(self.binding)

    def summary(self, dtype_size: int = 4) -> dict:
        e = [x.elements for x in self.entries]
        return {"entries": len(e), "total_elements": sum(e), "total_bytes": sum(e) * dtype_size,
                "max_elements": max(e, default=0), "min_elements": min(e, default=0)}

    def to_dict(self, dtype_size: int = 4) -> dict:
        return {"version": 1, "nest": self.nest, "binding": dict(self.binding),
                "dtype_size": dtype_size,
                "entries": [{"dependence": x.dep_id, "kind": x.kind, "array": x.array,
                             "variant": x.variant, "elements": x.elements,
                             "bytes": x.size_bytes(dtype_size)} for x in self.entries],
                "summary": self.summary(dtype_size)}


_KIND = {("read", "read"): "RAR", ("write", "read"): "RAW", ("read", "write"): "WAR",
         ("write", "write"): "WAW"}


# ----------------------------------------------------------------------------- enumeration
class _Trace:
    """Statement instances in schedule order with their references."""

    def __init__(self, nest: LoopNest, binding: Mapping[str, int], limit: int):
        if nest.has_kernel_call():
            nest = substitute_microkernel(nest)
        missing = [p for p in nest.params if p not in binding]
        if missing:
            raise UnboundParameterError(f"unbound parameters: {missing}")
        self.refs: dict = {}         # ref_id -> (label, array, kind)
        self.stmt_refs: dict = {}    # label -> [ref ids]
        self.stmt_iters: dict = {}   # label -> (iterator names)
        self.par_iters: dict = {}    # label -> parallel iterators (outer first)
        self.inst: list = []         # (label, counters tuple, {ref_id: element})
        self._limit = limit
        self._auto = 0
        self._labels: dict = {}      # id(StmtNode) -> label
        self._acc: dict = {}         # ref_id -> Access
        self._walk(nest.body, {p: int(binding[p]) for p in nest.params}, (), (), ())

    def _walk(self, nodes, env, iters, counters, pars):
        for n in nodes:
            if isinstance(n, LoopNode):
                lp = n.loop
                lo = lp.lower.eval(env)
                hi = min(u.eval(env) for u in lp.upper)
                c = 0
                for v in range(lo, hi, lp.step):
                    self._walk(n.body, {**env, lp.iterator: v}, iters + (lp.iterator,),
                               counters + (c,), pars + ((lp.iterator,) if lp.parallel else ()))
                    c += 1
                if hi <= lo:  # register the statements even if the loop is empty
                    self._register(n.body, iters + (lp.iterator,),
                                   pars + ((lp.iterator,) if lp.parallel else ()))
            elif isinstance(n, KernelRegion):
                self._walk(n.body, env, iters, counters, pars)
            elif isinstance(n, StmtNode):
                label = self._label(n, iters, pars)
                elems = {}
                for rid in self.stmt_refs[label]:
                    acc = self._acc[rid]
                    elems[rid] = tuple(ix.eval(env) for ix in acc.indices)
                self.inst.append((label, counters, elems))
                if len(self.inst) > self._limit:
                    raise WorkingSetError(f"more than {self._limit} statement instances; "
                                          "enumeration is for desk-size bindings")

    def _label(self, node, iters, pars):
        key = id(node)
        if key not in self._labels:
            st = node.stmt
            label = st.label or f"S{self._auto}"
            self._auto += 1
            self._labels[key] = label
            ids = []
            for k, acc in enumerate(st.read_accesses()):
                rid = f"{label}:r{k}"
                self.refs[rid] = (label, acc.array, "read")
                self._acc[rid] = acc
                ids.append(rid)
            rid = f"{label}:w0"
            self.refs[rid] = (label, st.target.array, "write")
            self._acc[rid] = st.target
            ids.append(rid)
            self.stmt_refs[label] = ids
            self.stmt_iters[label] = iters
            self.par_iters[label] = pars
        return self._labels[key]

    def _register(self, nodes, iters, pars):
        for n in nodes:
            if isinstance(n, LoopNode):
                self._register(n.body, iters + (n.loop.iterator,),
                               pars + ((n.loop.iterator,) if n.loop.parallel else ()))
            elif isinstance(n, KernelRegion):
                self._register(n.body, iters, pars)
            elif isinstance(n, StmtNode):
                self._label(n, iters, pars)

    def footprint(self, idxs) -> int:
        seen: dict = {}
        for i in idxs:
            _, _, elems = self.inst[i]
            for rid, e in elems.items():
                seen.setdefault(self.refs[rid][1], set()).add(e)
        return sum(len(v) for v in seen.values())


def working_sets(nest: LoopNest, binding: Mapping[str, int], sample_outer: bool = False,
                 limit: int = 2_000_000) -> WorkingSetReport:
    """Alg. 1 by enumeration: one WS_par or a (WS_min, WS_max) pair per dependence."""
    tr = _Trace(nest, binding, limit)
    inst = tr.inst
    by_label: dict = {}
    for i, (label, ctr, _) in enumerate(inst):
        by_label.setdefault(label, []).append(i)
    # element -> schedule positions, per reference
    pos: dict = {rid: {} for rid in tr.refs}
    for i, (_, _, elems) in enumerate(inst):
        for rid, e in elems.items():
            pos[rid].setdefault(e, []).append(i)
    entries = []
    arrays = sorted({a for _, a, _ in tr.refs.values()})
    for array in arrays:
        refs = [r for r in tr.refs if tr.refs[r][1] == array]
        for src in refs:
            for tgt in refs:
                s_label, _, s_kind = tr.refs[src]
                t_label, _, t_kind = tr.refs[tgt]
                kind = _KIND[(s_kind, t_kind)]
                # lexicographically first source instance with a later target
                src_i = None
                for i in by_label.get(s_label, []):
                    e = inst[i][2][src]
                    later = [t for t in pos[tgt].get(e, ()) if t > i]
                    if later:
                        src_i, targets = i, later
                        break
                if src_i is None:
                    continue
                dep_id = f"{src}->{tgt}"
                common = [p for p in tr.par_iters[s_label] if p in tr.par_iters[t_label]]
                if common and _spans(tr, pos, by_label, src, tgt, common):
                    # over the SOURCE statement's outermost parallel iterator, as the
                    # reference's classify_parallel_span reports it (depend.py:158-159)
                    ws = _par_footprint(tr, by_label, tr.par_iters[s_label][0], sample_outer)
                    entries.append(WorkingSetEntry(dep_id, kind, array, "par", ws))
                    continue
                key = lambda t: inst[t][1]  # counters: lexicographic order of iteration vectors
                tmin = min(targets, key=key)
                tmax = max(targets, key=key)
                ws_min = tr.footprint(range(src_i, tmin + 1))
                ws_max = tr.footprint(range(src_i, tmax + 1))
                if ws_min > ws_max:
                    raise WorkingSetError(f"WS_min {ws_min} > WS_max {ws_max} for {dep_id}")
                entries.append(WorkingSetEntry(dep_id, kind, array, "min", ws_min))
                entries.append(WorkingSetEntry(dep_id, kind, array, "max", ws_max))
    return WorkingSetReport(nest.name, tuple(sorted(binding.items())), tuple(entries))


def _spans(tr, pos, by_label, src, tgt, common) -> bool:
    s_label = tr.refs[src][0]
    t_label = tr.refs[tgt][0]
    s_it, t_it = tr.stmt_iters[s_label], tr.stmt_iters[t_label]
    for p in common:
        ps, pt = s_it.index(p), t_it.index(p)
        for i in by_label.get(s_label, []):
            e = tr.inst[i][2][src]
            for t in pos[tgt].get(e, ()):
                if t > i and tr.inst[i][1][ps] != tr.inst[t][1][pt]:
                    return True
    return False


def _par_footprint(tr, by_label, p, sample_outer) -> int:
    """Footprint across all values of the parallel loop with the outer
    iterators fixed at their lexicographic minimum (or also max / mid)."""
    def fixed(which) -> int:
        idxs = []
        for label, insts in by_label.items():
            iters = tr.stmt_iters[label]
            if p not in iters:
                continue
            k = iters.index(p)
            if k == 0:
                idxs.extend(insts)
                continue
            firsts = [tr.inst[i][1][:k] for i in insts]
            lo, hi = min(firsts), max(firsts)
            want = lo if which == "min" else hi if which == "max" else \
                tuple((a + b) // 2 for a, b in zip(lo, hi))
            idxs.extend(i for i in insts if tr.inst[i][1][:k] == want)
        return tr.footprint(idxs)

    best = fixed("min")
    if sample_outer:
        best = max(best, fixed("max"), fixed("mid"))
    return best


# ----------------------------------------------------------------------------- engine nest
def engine_gemm_nest(bm: int, bn: int, bk: int) -> str:
    """The tile engine's GEMM schedule as a `.pdl` nest (variants.emit_nest without
    split-K, tile sizes free so it can be enumerated at desk-size bindings): tile
    loops it, jt, kt, then the bm x bn x bk band."""
    return f"""param M, N, K;
array C[M][N];
array A[M][K];
array B[K][N];
gemm: parallel for (it = 0; it < M; it += {bm}) {{
  for (jt = 0; jt < N; jt += {bn}) {{
    for (kt = 0; kt < K; kt += {bk}) {{
      for (i = it; i < min(it + {bm}, M); i++) {{
        for (j = jt; j < min(jt + {bn}, N); j++) {{
          for (k = kt; k < min(kt + {bk}, K); k++) {{
            S: C[i][j] += A[i][k] * B[k][j];
          }}
        }}
      }}
    }}
  }}
}}
"""


def engine_gemm_working_sets(bm: int, bn: int, bk: int, M: int, N: int, K: int) -> WorkingSetReport:
    """Alg. 1's working sets of engine_gemm_nest in closed form (elements), valid when
    the tiles divide the extents and K >= 2 bk, N >= 2 bn:
      C (accumulator, RAR/RAW/WAR/WAW of C[i][j] across the k-blocks of its tile)
          WS_min = 5 (the next k step), WS_max = bm bn + (bm + bn)(K - bk) + 2 bk
          -- one TMEM accumulator + the tile's A and B panels (tile_working_sets'
          tmem.acc / 2 + l2.Apanel + l2.Bpanel) less the last k-block's panels;
      A (A[i][k] reused across j and the N-tiles) WS_min = 2 bk + 3,
          WS_max = bm K + (N - bn)(K + bm) + bk (bn - 1) + 1 + bn;
      B (B[k][j] reused across the parallel it loop) WS_par = MK + KN + MN.
    tests/test_rank.py checks these against the enumerated Alg. 1 (working_sets,
    itself pinned to the reference) at desk-size bindings."""
    c_max = bm * bn + (bm + bn) * (K - bk) + 2 * bk
    a_max = bm * K + (N - bn) * (K + bm) + bk * (bn - 1) + 1 + bn
    e = [WorkingSetEntry("S:r0->S:r0", "RAR", "A", "min", 2 * bk + 3),
         WorkingSetEntry("S:r0->S:r0", "RAR", "A", "max", a_max),
         WorkingSetEntry("S:r1->S:r1", "RAR", "B", "par", M * K + K * N + M * N)]
    for dep, kind in (("S:r2->S:r2", "RAR"), ("S:r2->S:w0", "WAR"), ("S:w0->S:r2", "RAW"),
                      ("S:w0->S:w0", "WAW")):
        e += [WorkingSetEntry(dep, kind, "C", "min", 5), WorkingSetEntry(dep, kind, "C", "max", c_max)]
    return WorkingSetReport("gemm", (("K", K), ("M", M), ("N", N)), tuple(e))


# ----------------------------------------------------------------------------- tile form
def tile_working_sets(layer, variant, n_images: int, sms: int = 148) -> WorkingSetReport:
    """Closed-form working sets of one tile-engine schedule on one SM.

    `layer`: workloads.ConvLayer; `variant`: variants.TileVariant.  Elements
    are fp32 words.  Entries:
      smem.A / smem.B      pipeline stages of activation / weight tiles
      tmem.acc / tmem.A    accumulator ping-pong and TMEM-staged A slots
      l2.wslice            weights of the N-tile, reused by every M-tile
      l2.halo              input rows shared by vertically adjacent pixel tiles
                           running concurrently (3x3 taps)
      mem.stream           compulsory x / w / y traffic per SM
    """
    from .variants import _is_gemm, engine_geometry
    g = engine_geometry(layer, variant, n_images)
    planes = 2 if variant.mode == "3xtf32" else 1
    ks = g["ks"]
    e = []
    if _is_gemm(layer):
        e.append(WorkingSetEntry("smem.A", "buffer", "A", "smem", g["stages"] * 128 * ks))
        e.append(WorkingSetEntry("smem.B", "buffer", "B", "smem", g["stages"] * variant.bn * ks * planes))
        e.append(WorkingSetEntry("tmem.acc", "buffer", "C", "tmem", 2 * 128 * variant.bn))
        if g["tslots"]:
            e.append(WorkingSetEntry("tmem.A", "buffer", "A", "tmem", g["tslots"] * 128 * ks * planes))
        e.append(WorkingSetEntry("l2.Bpanel", "reuse", "B", "l2", layer.K * variant.bn))
        e.append(WorkingSetEntry("l2.Apanel", "reuse", "A", "l2", 128 * layer.K))
        e.append(WorkingSetEntry("mem.stream", "stream", "ABC", "mem",
                                 int(layer.bytes() // 4 // sms)))
        return WorkingSetReport(layer.name(), (("variant", variant.vid),), tuple(e))
    e.append(WorkingSetEntry("smem.A", "buffer", "x", "smem", g["stages"] * 128 * ks))
    e.append(WorkingSetEntry("smem.B", "buffer", "w", "smem",
                             g["stages"] * variant.bn * ks * planes))
    e.append(WorkingSetEntry("tmem.acc", "buffer", "y", "tmem", 2 * 128 * variant.bn))
    if g["tslots"]:
        e.append(WorkingSetEntry("tmem.A", "buffer", "x", "tmem", g["tslots"] * 128 * ks * planes))
    e.append(WorkingSetEntry("l2.wslice", "reuse", "w", "l2",
                             layer.C_alloc * layer.R * layer.S * variant.bn * planes))
    if layer.R > 1:
        rows = min(g["tiles_concurrent"], g["m_tiles"]) * g["tile_rows_in"]
        e.append(WorkingSetEntry("l2.halo", "reuse", "x", "l2", rows * layer.W * layer.C_alloc))
    stream = (layer.x_touched(n_images) + layer.K * layer.C * layer.R * layer.S
              + n_images * layer.K * layer.P * layer.Q) // sms
    e.append(WorkingSetEntry("mem.stream", "stream", "xwy", "mem", int(stream)))
    return WorkingSetReport(layer.name(), (("N", n_images), ("variant", variant.vid)), tuple(e))
