"""One profiled launch per GEMM shape of the BASELINE sweep (and PR1), for
`ncu --profile-from-start off`: each shape is warmed up outside the profiler
range, then launched once inside it.

    ncu --profile-from-start off --metrics ... -o out python scripts/ncu_gemm_case.py [mode]
"""
import sys

sys.path.insert(0, ".")
import torch

import paper_2006_02230_b200 as P
from paper_2006_02230_b200 import workloads as W

mode = sys.argv[1] if len(sys.argv) > 1 else "3xtf32"
torch.manual_seed(0)
for (m, n, k) in W.GEMM_SWEEP:
    a = torch.rand((m, k), device="cuda") * 2 - 1
    b = torch.rand((k, n), device="cuda") * 2 - 1
    c = torch.empty((m, n), device="cuda")
    for _ in range(3):
        P.gemm(a, b, c, mode=mode)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    P.gemm(a, b, c, mode=mode)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("gemm", m, n, k, flush=True)
# PR1 (BASELINE configs[0]): one image, 64 -> 64 channels, 56x56, 3x3
layer = W.PR1 if hasattr(W, "PR1") else W.ConvLayer(0, 64, 64, 56, 3, 1)
x = torch.rand((1, layer.C_alloc // 16, layer.H, layer.W, 16), device="cuda")
w = torch.rand((layer.K // 16, layer.C_alloc // 16, layer.R, layer.S, 16, 16), device="cuda")
bias = torch.rand(layer.K, device="cuda")
pw = P.prepack_weights(w, mode=mode, channels=layer.C)
y = torch.empty((1, layer.K // 16, layer.P, layer.Q, 16), device="cuda")
for _ in range(3):
    P.conv2d_nchw16c(x, pw, bias, stride=layer.stride, pad=layer.pad, relu=True, mode=mode, out=y)
torch.cuda.synchronize()
torch.cuda.profiler.start()
P.conv2d_nchw16c(x, pw, bias, stride=layer.stride, pad=layer.pad, relu=True, mode=mode, out=y)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("pr1", flush=True)
