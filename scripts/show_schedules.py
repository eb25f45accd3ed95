"""Print the library's schedule for every ResNet-50 layer: new box search vs the round-1
single-image geometry (PDL_RASTER_SINGLE_IMAGE_TILES).  Host-only."""
import sys
sys.path.insert(0, '.')
from paper_2006_02230_b200 import _lib, workloads as W
f = lambda s: (s['tile_w'], s['tile_h'], s['tile_images'], s['m_tiles'], s['n_tiles'], s['split'], s['halo'], s['seg_rows'], s['flat'])
for flags, mname in ((0, "3xtf32"), (16, "tf32")):
    for n in (256, 32, 28):
        tn = to = 0
        for l in W.LAYERS:
            s = _lib.conv_schedule(n, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, flags)
            o = _lib.conv_schedule(n, l.C, l.K, l.H, l.W, l.R, l.S, l.stride, l.pad, flags, cfg={"raster": 8})
            print(mname, n, l.name(), f(s), f(o), "" if f(s) == f(o) else f"tiles x{s['m_tiles']/o['m_tiles']:.3f}")
