"""Schedule variants of the B200 tile engine (SPEC `variants` module,
SPEC.md:468-529, re-targeted).

On the CPU a variant is a tiled / interchanged loop nest emitted as C.  On the
B200 the loop nest is fixed (the persistent tile engine), and what varies is
the tile configuration a `pdl_tile_cfg` carries:

  bn       output channels (conv K / GEMM N) per CTA tile: 64 | 128 | 256 (TF32 only:
           one accumulation segment per tile, streaming epilogue)
  bk       reduction elements per pipeline stage: 16 * cg, cg in {1, 2, 4}
  cluster  CTAs sharing (multicasting) each weight tile: 1 | 2 | 4
  mode     "3xtf32" | "tf32"

`generate_variants` enumerates the legal ones deterministically (ids sorted,
deduplicated), `legality_check` runs a variant against the default schedule on
the GPU (interpreter-equivalence in the SPEC's sense, at the mode's tolerance:
variants with the same bk and segmenting reduce every element in the same order
and agree bitwise; a different bk re-associates the channel/tap sum inside a
256-element accumulation segment, and 256-column tiles sum the whole reduction in
one segment), `emit_launch` is the B200 analogue of
`emit_c`: the launch configuration (a dict accepted as `cfg=` by the ops).
`engine_geometry` restates the host's tiling rules (csrc/pdl_capi.cu) so the
analytical ranker can reason about a variant without launching it.
"""
from __future__ import annotations

from dataclasses import dataclass, field

# kernel instances compiled into libpdl.so (csrc/pdl_capi.cu dispatch_bn)
_CONV_INSTANCES = {(64, 1), (64, 2), (64, 4), (128, 1), (128, 2)}
_SMEM_BUDGET = 216 * 1024
_SEG_ELEMS = 256


@dataclass(frozen=True, order=True)
class TileVariant:
    vid: str
    bn: int
    bk: int
    cluster: int
    mode: str = "3xtf32"

    @property
    def cg(self) -> int:
        return self.bk // 16


@dataclass
class VariantConfig:
    bn_menu: tuple = (64, 128, 256)
    cg_menu: tuple = (1, 2, 4)
    cluster_menu: tuple = (1, 2, 4)
    modes: tuple = ("3xtf32",)
    cap: int = 64


def _is_gemm(layer) -> bool:
    return hasattr(layer, "M") and not hasattr(layer, "R")


def _is_stem(layer) -> bool:
    return not _is_gemm(layer) and layer.C <= 4 and layer.S <= 8 and layer.R <= 7


def legal(layer, v: TileVariant) -> bool:
    """Static legality: a compiled instance exists, channel grouping matches
    the packed weight rows, the stage fits shared memory / TMEM."""
    if _is_gemm(layer):
        # GEMM instances: bn in {64, 128}, bk = 32, cluster in {1, 2, 4}
        return v.bk == 32 and v.bn in (64, 128) and v.cluster in (1, 2, 4) and \
            not (v.bn > 64 and layer.N <= 64)
    if _is_stem(layer):
        return v.bn == 64 and v.cluster == 1 and v.bk == 32
    ct = (layer.C + 15) // 16
    if v.bn == 256:
        # TF32 instance only, whole 256-column slices, no cluster (conv_default_cfg)
        if not (v.mode == "tf32" and v.cg == 2 and v.cluster == 1 and layer.K % 256 == 0):
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
    tslots = min(8, (512 - 2 * v.bn) // slot) if v.mode == "3xtf32" else 0
    return {"stage_bytes": stage, "stages": stages, "ks": ks, "tslots": tslots}


def stem_tile(layer) -> tuple:
    """BW x BH output-pixel tile of the narrow-channel stem (conv_fwd_stem in
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


def engine_geometry(layer, v: TileVariant, n_images: int, sms: int = 148) -> dict:
    """Tile geometry the host code picks (conv_geom in csrc/pdl_capi.cu)."""
    g = stage_sizes(v)
    if _is_gemm(layer):
        m_tiles, n_tiles = -(-layer.M // 128), -(-layer.N // v.bn)
        g.update(flat=True, bw=128, bh=1, bni=1, rows_valid=min(layer.M, 128), m_eff=1.0,
                 m_tiles=m_tiles, n_tiles=n_tiles, tiles=m_tiles * n_tiles,
                 num_kb=-(-layer.K // 32), seg_kb=max(1, _SEG_ELEMS // 32),
                 tiles_concurrent=sms, tile_rows_in=1)
        return g
    P, Q = layer.P, layer.Q
    flat = layer.R == 1 and layer.S == 1 and layer.stride == 1 and layer.pad == 0
    Pg, Qg = (1, P * Q) if flat else (P, Q)
    if _is_stem(layer):
        bw, bh = stem_tile(layer)
        bni = 1
    else:
        bw = min(Qg, 128)
        bh = min(Pg, 128 // bw)
        bni = max(1, min(n_images, 128 // (bw * bh))) if bh == Pg else 1
    tiles_w, tiles_h = -(-Qg // bw), -(-Pg // bh)
    m_tiles = tiles_w * tiles_h * -(-n_images // bni)
    n_tiles = -(-layer.K // v.bn)
    rows = bw * bh * bni
    num_kb = layer.R if _is_stem(layer) else ((layer.C_alloc // 16) // v.cg) * layer.R * layer.S
    g.update(flat=flat, bw=bw, bh=bh, bni=bni, rows_valid=rows, m_eff=rows / 128.0,
             m_tiles=m_tiles, n_tiles=n_tiles, tiles=m_tiles * n_tiles, num_kb=num_kb,
             seg_kb=num_kb if v.bn > 128 else max(1, _SEG_ELEMS // g["ks"]), tiles_concurrent=sms,
             tile_rows_in=(bh - 1) * layer.stride + layer.R)
    return g


def generate_variants(layer, cfg: VariantConfig = VariantConfig()) -> list:
    """All legal tile configurations of a conv layer, deterministic order."""
    out = {}
    for mode in cfg.modes:
        for bn in cfg.bn_menu:
            for cg in ((2,) if _is_gemm(layer) else cfg.cg_menu):
                for cl in cfg.cluster_menu:
                    v = TileVariant(f"bn{bn}_bk{16 * cg}_c{cl}_{mode}", bn, 16 * cg, cl, mode)
                    if legal(layer, v):
                        out[v.vid] = v
    vs = [out[k] for k in sorted(out)]
    if not vs:
        import warnings
        warnings.warn(f"no legal variant for {layer.name()}; using the default only")
    if len(vs) > cfg.cap:
        import warnings
        warnings.warn(f"{len(vs)} variants for {layer.name()}; keeping the first {cfg.cap}")
    return vs[:cfg.cap]


def emit_launch(v: TileVariant) -> dict:
    """Launch configuration for the ops (`cfg=`), the B200 analogue of emit_c:
    the fields of `pdl_tile_cfg` (include/pdl.h)."""
    return {"bm": 128, "bn": v.bn, "bk": v.bk, "cluster_m": v.cluster}


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
