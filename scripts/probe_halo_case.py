"""Debug: halo vs per-tap boxes on one shape, repeated, vs the fp64 oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

C, K, H, R, N = 48, 32, 9, 3, 3
layer = W.ConvLayer(0, C, K, H, R, 1)
x, w, b = W.conv_inputs(layer, N, seed=31)
pw = P.prepack_weights(torch.from_numpy(w).cuda())
xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
ref = oracle.conv2d_f64(x, w, b, stride=1, pad=1, relu=True)
for split in (1, 2, 3):
    for name, raster in (("halo", 0), ("taps", 16)):
        outs = [P.conv2d_nchw16c(xd, pw, bd, stride=1, pad=1, relu=True,
                                 cfg={"split_k": split, "cluster_m": 1, "raster": raster}).cpu().numpy()
                for _ in range(4)]
        same = all(np.array_equal(outs[0], o) for o in outs[1:])
        errs = [float(np.abs(o - ref).max() / np.abs(ref).max()) for o in outs]
        bad = np.argwhere(np.abs(outs[0] - ref) > 1e-4 * np.abs(ref).max())
        print(f"split {split} {name}: deterministic={same} rel={['%.1e' % e for e in errs]} bad={bad[:4].tolist()}",
              flush=True)
