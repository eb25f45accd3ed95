"""Schedule variants of the B200 tile engine (SPEC `variants` module,
SPEC.md:468-529, re-targeted).

On the CPU a variant is a tiled / interchanged loop nest with one loop marked
parallel, emitted as C.  On the B200 the engine executes the Fig. 9 / Fig. 1 nest
as a persistent implicit GEMM, and the same three transformation families become
the fields of a `pdl_tile_cfg`:

  tiling        bn      output channels (conv K / GEMM N) per CTA tile: 64 | 128 |
                        256 (TF32 only: one accumulation segment, streaming epilogue)
                bk      reduction elements per k-block: 16 * cg, cg in {1, 2, 4}
                seg     output-pixel tile shape: box tiles ("off") or segment tiles
                        spanning images ("on"; small 1x1 maps), "auto" = library rule
                halo    stride-1 spatial convs: the tile's input halo loaded once per
                        channel group ("on") or one A box per tap ("off")
  interchange   order   tile loop order: output-channel tiles fastest ("n": CTAs
                        running together share activation rows) or output-pixel tiles
                        fastest ("m": they share a weight slice)
  parallel loop split   the reduction loop split across CTAs (split-K): 1 = the tile
                        loops alone are parallel; k > 1 = the reduction loop too, in k
                        ranges; 0 = library planner (only with sub-wave tile counts)
                cluster CTAs sharing (multicasting) each weight tile: 1 | 2 | 4

`generate_variants(nest, cfg, binding)` takes the `.pdl` LoopNest (the conv /
GEMM nest is recognised by the executor's matcher) or an already
recognised layer shape, enumerates the menus, and keeps one variant per distinct
EFFECTIVE schedule: every candidate is run through the library's own planner
(`pdl_conv2d_schedule` / `pdl_gemm_schedule`, host-only) so that a request the
engine would silently override (halo on a 1x1 layer, a split on a full wave,
segment tiles on an odd-width map) does not appear as a separate variant.  Ids are
deterministic (sorted); the first id per schedule wins.  `legality_check` runs a
variant against the default schedule on the GPU (interpreter equivalence at the
mode tolerance); `emit_launch` is the B200 analogue of `emit_c`: the launch
configuration (a dict accepted as `cfg=` by the ops); `emit_nest` writes the
variant's tiled loop nest as `.pdl` text (provenance, parseable).
"""
from __future__ import annotations

from dataclasses import dataclass

# kernel instances compiled into libpdl.so (csrc/pdl_capi.cu dispatch_bn)
_CONV_INSTANCES = {(64, 1), (64, 2), (64, 4), (128, 1), (128, 2)}
_SMEM_BUDGET = 216 * 1024
_SEG_ELEMS = 256
_SMS = 148

# include/pdl.h raster bits
RASTER_M_FASTEST, RASTER_BOX_TILES, RASTER_SEG_TILES, RASTER_NO_HALO, RASTER_HALO_CG4 = 1, 2, 4, 16, 64
RASTER_SINGLE_IMAGE_TILES = 8


@dataclass(frozen=True, order=True)
class TileVariant:
    vid: str
    bn: int
    bk: int
    cluster: int
    mode: str = "3xtf32"
    order: str = "n"      # "n": output-channel tiles fastest, "m": output-pixel tiles fastest
    halo: str = "auto"    # "on" | "off" | "auto"
    seg: str = "auto"     # "on" | "off" | "auto"
    split: int = 0        # 0: library planner, 1: no split, k: k reduction ranges
    tile: str = "auto"    # "auto": the library's box search over (pixels wide, pixels high, images);
                          # "single": a tile holds several images only when a whole image fits;
                          # "WxHxN": that box (PDL_RASTER_TILE)

    @property
    def cg(self) -> int:
        return self.bk // 16

    def provenance(self) -> dict:
        return {"bn": self.bn, "bk": self.bk, "cluster": self.cluster, "mode": self.mode,
                "order": self.order, "halo": self.halo, "seg": self.seg, "split": self.split,
                "tile": self.tile}


def make_variant(bn: int, bk: int, cluster: int, mode: str = "3xtf32", order: str = "n",
                 halo: str = "auto", seg: str = "auto", split: int = 0, tile: str = "auto") -> TileVariant:
    """Variant with its canonical id (defaults leave no suffix, so the ids of the
    round-1 bn x bk x cluster menu are unchanged)."""
    vid = f"bn{bn}_bk{bk}_c{cluster}_{mode}"
    if order == "m":
        vid += "_om"
    if halo != "auto":
        vid += "_h1" if halo == "on" else "_h0"
    if seg != "auto":
        vid += "_s1" if seg == "on" else "_s0"
    if split:
        vid += f"_k{split}"
    if tile != "auto":
        vid += "_t1" if tile == "single" else f"_t{tile}"
    return TileVariant(vid, bn, bk, cluster, mode, order, halo, seg, split, tile)


def variant_from_record(vid: str, rec: dict, mode: str) -> TileVariant:
    """Rebuild a variant from a sweep record (scripts/sweep_variants.py)."""
    return TileVariant(vid, rec["bn"], rec["bk"], rec["cluster"], mode, rec.get("order", "n"),
                       rec.get("halo", "auto"), rec.get("seg", "auto"), rec.get("split", 0),
                       rec.get("tile", "auto"))


@dataclass
class VariantConfig:
    bn_menu: tuple = (64, 128, 256)
    cg_menu: tuple = (1, 2, 4)
    cluster_menu: tuple = (1, 2, 4)
    modes: tuple = ("3xtf32",)
    order_menu: tuple = ("n", "m")
    halo_menu: tuple = ("auto", "on", "off")
    seg_menu: tuple = ("auto", "on", "off")
    split_menu: tuple = (0, 1, 2, 3, 4, 6, 8)   # used only when the tiles leave SMs idle
    tile_menu: tuple = ("auto", "single")
    cap: int = 256


def _is_gemm(layer) -> bool:
    return hasattr(layer, "M") and not hasattr(layer, "R")


def _is_stem(layer) -> bool:
    return not _is_gemm(layer) and layer.C <= 4 and layer.S <= 8 and layer.R <= 7


def _mode_flags(mode: str) -> int:
    from ._lib import MODES
    return MODES[mode]


def legal(layer, v: TileVariant) -> bool:
    """Static legality: a compiled instance exists, channel grouping matches
    the packed weight rows, the stage fits shared memory / TMEM."""
    if _is_gemm(layer):
        # GEMM instances: bn in {64, 128}, bk = 32, cluster in {1, 2, 4}
        return v.bk == 32 and v.bn in (64, 128) and v.cluster in (1, 2, 4) and \
            not (v.bn > 64 and layer.N <= 64) and v.halo == "auto" and v.seg == "auto" and v.tile == "auto"
    if _is_stem(layer):
        return v.bn == 64 and v.cluster == 1 and v.bk == 32 and v.order == "n" and \
            v.halo == "auto" and v.seg == "auto" and v.split in (0, 1) and v.tile == "auto"
    ct = (layer.C + 15) // 16
    if v.bn == 256:
        # whole 256-column slices, no cluster / split; TF32: bk 32 / 64, 3xTF32: bk 32 (one accumulator)
        if not (v.cg in ((2, 4) if v.mode == "tf32" else (2,)) and v.cluster == 1 and layer.K % 256 == 0 and
                v.split in (0, 1)):
            return False
    elif (v.bn, v.cg) not in _CONV_INSTANCES and not (v.mode == "tf32" and (v.bn, v.cg) == (128, 4)):
        return False
    if ct % v.cg:
        return False
    if (ct % 2 == 0) != (v.cg >= 2):        # 128-byte weight rows need cg >= 2
        return False
    if v.bn % (8 * v.cluster):
        return False
    if v.bn > 64 and layer.K <= 64:
        return False
    if v.cluster > 1 and (v.order == "m" or v.halo == "on"):
        return False                        # tile order / halo need cluster 1
    g = stage_sizes(v)
    return g["stages"] >= 2 and (v.mode != "3xtf32" or g["tslots"] >= 2)


def stage_sizes(v: TileVariant) -> dict:
    planes = 2 if v.mode == "3xtf32" else 1
    a_bytes = v.cg * 128 * 64
    b_bytes = v.bn * 64 * v.cg
    stage = a_bytes + b_bytes * planes
    stages = min(16, _SMEM_BUDGET // stage)
    ks = 16 * v.cg
    slot = (2 * ks) if v.mode == "3xtf32" else ks
    acc_cols = v.bn if v.bn > 128 else 2 * v.bn  # 3xTF32 at 256 columns: a single accumulator
    tslots = min(8, (512 - acc_cols) // slot) if v.mode == "3xtf32" else 0
    return {"stage_bytes": stage, "stages": stages, "ks": ks, "tslots": tslots}


def emit_launch(v: TileVariant) -> dict:
    """Launch configuration for the ops (`cfg=`), the B200 analogue of emit_c:
    the fields of `pdl_tile_cfg` (include/pdl.h)."""
    raster = 0
    if v.order == "m":
        raster |= RASTER_M_FASTEST
    if v.halo == "off":
        raster |= RASTER_NO_HALO
    elif v.halo == "on" and v.cg == 4 and v.mode == "3xtf32":
        raster |= RASTER_HALO_CG4
    if v.seg == "off":
        raster |= RASTER_BOX_TILES
    elif v.seg == "on":
        raster |= RASTER_SEG_TILES
    if v.tile == "single":
        raster |= RASTER_SINGLE_IMAGE_TILES
    elif v.tile != "auto":
        bw, bh, bni = (int(t) for t in v.tile.split("x"))
        raster |= bw << 8 | bh << 16 | bni << 24
    cfg = {"bm": 128, "bn": v.bn, "bk": v.bk, "cluster_m": v.cluster}
    if raster:
        cfg["raster"] = raster
    if v.split:
        cfg["split_k"] = v.split
    return cfg


def schedule(layer, v: TileVariant, n_images: int) -> dict:
    """The schedule libpdl will actually run for this variant (pdl_conv2d_schedule /
    pdl_gemm_schedule; host-only, no GPU needed)."""
    from ._lib import conv_schedule, gemm_schedule
    if _is_gemm(layer):
        return gemm_schedule(layer.M, layer.N, layer.K, _mode_flags(v.mode), emit_launch(v))
    return conv_schedule(n_images, layer.C, layer.K, layer.H, layer.W, layer.R, layer.S, layer.stride,
                         layer.pad, _mode_flags(v.mode), emit_launch(v))


def _signature(sched: dict, v: TileVariant) -> tuple:
    keys = ("kind", "bn", "bk", "cluster", "tile_w", "tile_h", "tile_images", "seg_rows", "m_tiles",
            "n_tiles", "split", "kb_per", "halo", "resident", "pair", "order")
    return (v.mode,) + tuple(sched[k] for k in keys)


def stem_tile(layer) -> tuple:
    """BW x BH output-pixel tile of the narrow-channel stem (stem_tile in
    csrc/pdl_capi.cu): its input halo is one TMA box / pipeline stage."""
    P, Q, s, R, S = layer.P, layer.Q, layer.stride, layer.R, layer.S
    best, pick = float("inf"), None
    for bw in range(min(Q, 128), 0, -1):
        bh = min(P, 128 // bw)
        bxw, bxh = (bw - 1) * s + S, (bh - 1) * s + R
        if bxw > 256 or bxh > 256 or 16 * bxw * bxh > 16384:
            continue
        tiles = -(-Q // bw) * -(-P // bh)
        cost = tiles * max(R * 700.0, 4.4 * bxw * bxh)
        if cost < best - 1e-9:
            best, pick = cost, (bw, bh)
    return pick


def engine_geometry(layer, v: TileVariant, n_images: int, sms: int = _SMS) -> dict:
    """Tile geometry of the schedule the library runs (from its own planner)."""
    g = stage_sizes(v)
    s = schedule(layer, v, n_images)
    rows = s["tile_w"] * s["tile_h"] * (1 if s["seg_rows"] else s["tile_images"])
    g.update(s)
    g.update(bw=s["tile_w"], bh=s["tile_h"], bni=s["tile_images"], rows_valid=min(rows, 128),
             m_eff=min(rows, 128) / 128.0, tiles=s["m_tiles"] * s["n_tiles"],
             units=s["m_tiles"] * s["n_tiles"] * max(1, s["split"]),
             seg_kb=s["num_kb"] if s["bn"] > 128 else max(1, _SEG_ELEMS // max(g["ks"], 1)),
             tiles_concurrent=sms, ks=(s["bk"] if not _is_gemm(layer) else 32),
             tile_rows_in=1 if _is_gemm(layer) else (s["tile_h"] - 1) * layer.stride + layer.R,
             flat=bool(s["flat"]))
    return g


def _shape_of(nest, binding):
    """(layer shape, images) of a conv / GEMM LoopNest, via the executor's matcher."""
    from .executor import ConvPlan, GemmPlan, plan_program
    from .workloads import ConvShape, GemmShape
    plans = plan_program([nest], binding)
    heavy = [p for p in plans if isinstance(p, (ConvPlan, GemmPlan))]
    if len(heavy) != 1:
        raise ValueError("generate_variants: the nest is not one conv / GEMM")
    p = heavy[0]
    if isinstance(p, GemmPlan):
        return GemmShape(p.M, p.N, p.K), 1
    # the nest's input is pre-padded (Fig. 9); the B200 call takes it unpadded with pad 0
    return ConvShape(p.CT * 16, p.KT * 16, p.Hp, p.Wp, p.R, p.S, p.stride, 0), p.N


def generate_variants(nest_or_layer, cfg: VariantConfig = VariantConfig(), binding=None,
                      n_images: int | None = None) -> list:
    """All legal, distinct schedules of a conv / GEMM, deterministic id order.

    `nest_or_layer`: a LoopNest (with `binding`) -- SPEC.md:483's signature -- or a
    layer shape (workloads.ConvLayer / ConvShape / GemmShape).  `n_images` (taken
    from the nest when given one) decides whether split-K candidates exist: they do
    only when the unsplit tiles leave SMs idle."""
    from .loopnest import LoopNest
    if isinstance(nest_or_layer, LoopNest):
        if binding is None:
            raise ValueError("generate_variants(nest): a parameter binding is required")
        layer, n = _shape_of(nest_or_layer, binding)
        n_images = n if n_images is None else n_images
    else:
        layer = nest_or_layer
    n = 256 if n_images is None else n_images
    gemm, stem = _is_gemm(layer), _is_stem(layer)
    seen: dict = {}
    for mode in cfg.modes:
        for bn in cfg.bn_menu:
            for cg in ((2,) if gemm else cfg.cg_menu):
                for cl in cfg.cluster_menu:
                    v0 = make_variant(bn, 16 * cg, cl, mode)
                    if not legal(layer, v0):
                        continue
                    try:
                        s0 = schedule(layer, v0, n)
                    except Exception:  # noqa: BLE001 -- the planner refused the combination
                        continue
                    sub_wave = s0["m_tiles"] * s0["n_tiles"] < _SMS and n_images is not None
                    splits = cfg.split_menu if sub_wave else (0,)
                    for order in (cfg.order_menu if cl == 1 else ("n",)):
                        for halo in (("auto",) if gemm or stem else cfg.halo_menu):
                            for seg in (("auto",) if gemm or stem else cfg.seg_menu):
                                for sp in splits:
                                    for tile in (("auto",) if gemm or stem else cfg.tile_menu):
                                        v = make_variant(bn, 16 * cg, cl, mode, order, halo, seg, sp, tile)
                                        if not legal(layer, v):
                                            continue
                                        try:
                                            sig = _signature(schedule(layer, v, n), v)
                                        except Exception:  # noqa: BLE001
                                            continue
                                        if sig not in seen or v.vid < seen[sig].vid:
                                            seen[sig] = v
    vs = sorted(seen.values(), key=lambda v: v.vid)
    if not vs:
        import warnings
        warnings.warn(f"no legal variant for {layer.name()}; using the default only")
    if len(vs) > cfg.cap:
        import warnings
        warnings.warn(f"{len(vs)} variants for {layer.name()}; keeping the first {cfg.cap}")
    return vs[:cfg.cap]


def emit_nest(layer, v: TileVariant, n_images: int = 1) -> str:
    """The variant as a transformed loop nest (SPEC `Variant.nest`), `.pdl` text.

    GEMM: the Fig. 1 nest tiled the way the engine runs it -- the two tile loops in
    the variant's order (the outer one `parallel`), the reduction cut into the
    split-K ranges and k-blocks, and the 128 x bn x 32 microkernel band innermost.
    It parses with loopnest.parse and is interpreter-equivalent to Fig. 1 (the
    reduction is only re-associated).  Conv: a one-line provenance comment of the
    effective schedule (its tile shapes -- segment tiles spanning images, halo
    reuse -- are not loop tilings of the Fig. 9 nest)."""
    s = schedule(layer, v, n_images)
    if not _is_gemm(layer):
        tiles = "pixel tiles" if not s["seg_rows"] else f"segment tiles of {s['seg_rows']} rows"
        return (f"// {layer.name()} x{n_images} {v.vid}: {s['m_tiles']} {tiles} "
                f"({s['tile_w']}x{s['tile_h']}x{s['tile_images']}) x {s['n_tiles']} channel tiles of "
                f"{s['bn']}; {s['num_kb']} k-blocks of {s['bk']} in {s['split']} range(s) of "
                f"{s['kb_per']}; halo {'on' if s['halo'] else 'off'}; resident weights "
                f"{'on' if s['resident'] else 'off'}; "
                f"{'pixel' if s['order'] else 'channel'}-tiles fastest\n")
    bn, kr = s["bn"], s["kb_per"] * 32
    loops = [("it", "M", 128), ("jt", "N", bn)]
    if s["order"] == 1:
        loops.reverse()
    (o1, e1, t1), (o2, e2, t2) = loops
    lines = ["param M, N, K;", "array C[M][N];", "array A[M][K];", "array B[K][N];",
             f"gemm: parallel for ({o1} = 0; {o1} < {e1}; {o1} += {t1}) {{",
             f"  for ({o2} = 0; {o2} < {e2}; {o2} += {t2}) {{",
             f"    for (kr = 0; kr < K; kr += {kr}) {{",
             "      for (kt = kr; kt < min(kr + %d, K); kt += 32) {" % kr,
             "        for (i = it; i < min(it + 128, M); i++) {",
             f"          for (j = jt; j < min(jt + {bn}, N); j++) {{",
             "            for (k = kt; k < min(kt + 32, K); k++) {",
             "              S: C[i][j] += A[i][k] * B[k][j];",
             "            }", "          }", "        }", "      }", "    }", "  }", "}"]
    return "\n".join(lines) + "\n"


MODE_TOLERANCE = {"3xtf32": 1e-5, "tf32": 1e-2}


def legality_check(layer, v: TileVariant, n_images: int = 2, seed: int = 0,
                   return_detail: bool = False):
    """Run the variant and the library default on the same inputs on the GPU.
    Legal iff finite and max|got - ref| <= tol(mode) * max|ref|; the detail
    reports whether the two were bitwise equal."""
    import numpy as np
    import torch
    from . import ops
    from .workloads import conv_inputs
    x, w, b = conv_inputs(layer, n_images, seed=seed)
    X, Wt, B = (torch.from_numpy(t).cuda() for t in (x, w, b))
    ref = ops.conv2d_nchw16c(X, Wt, B, stride=layer.stride, pad=layer.pad, relu=True,
                             mode=v.mode, channels=layer.C)
    got = ops.conv2d_nchw16c(X, Wt, B, stride=layer.stride, pad=layer.pad, relu=True,
                             mode=v.mode, channels=layer.C, cfg=emit_launch(v))
    bitwise = bool(torch.equal(ref, got))
    scale = float(ref.abs().max()) or 1.0
    rel = float((got - ref).abs().max()) / scale
    ok = bool(np.isfinite(got.cpu().numpy()).all()) and rel <= MODE_TOLERANCE[v.mode]
    return (ok, {"bitwise": bitwise, "max_rel": rel}) if return_detail else ok


__all__ = ["TileVariant", "VariantConfig", "make_variant", "variant_from_record", "legal", "stage_sizes",
           "emit_launch", "schedule", "engine_geometry", "generate_variants", "emit_nest",
           "legality_check", "MODE_TOLERANCE", "stem_tile"]
