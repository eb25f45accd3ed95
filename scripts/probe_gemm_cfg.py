"""Correctness of GEMM schedules (bn, split_k, cluster_m) against fp64."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle
import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

for (m, n, k) in [(1024, 1024, 1024), (512, 512, 512), (256, 192, 2048)]:
    a, b = W.gemm_inputs(m, n, k, seed=2)
    ref = oracle.gemm_f64(a, b)
    for bn in (64, 128):
        for sk in (1, 2, 3):
            for cl in (1, 2):
                c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                           cfg={"bn": bn, "split_k": sk, "cluster_m": cl}).cpu().numpy()
                err = np.abs(c - ref).max() / np.abs(ref).max()
                bad = np.argwhere(np.abs(c - ref) > 1e-3 * np.abs(ref).max())
                rows = sorted({int(r) // 128 for r, _ in bad})[:8]
                cols = sorted({int(cc) // 64 for _, cc in bad})[:8]
                print(f"{m}x{n}x{k} bn={bn} split={sk} cl={cl}: rel {err:.2e}  bad m-tiles {rows} n64-tiles {cols}",
                      flush=True)
