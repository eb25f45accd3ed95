"""One small launch per kernel family, for compute-sanitizer (tests/test_gpu_sanitizer.py):

    compute-sanitizer --tool memcheck|racecheck|synccheck --error-exitcode 99 \
        python scripts/sanitize_case.py FAMILY

FAMILY: stem | halo | resident | splitk | gemm | gemm_splitk | host | simt | layout.
Each case also checks its result against the float64 oracle (exit 1 on mismatch),
so a run that passes the sanitizer is known to have computed the right thing.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_2006_02230_b200 as P  # noqa: E402
from paper_2006_02230_b200 import workloads as W  # noqa: E402


def rel(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30))


def conv_case(layer, n, cfg=None, host=False):
    x, w, b = W.conv_inputs(layer, n, seed=3)
    pw = P.prepack_weights(torch.from_numpy(w).cuda(), channels=layer.C)
    if host:
        y = P.conv2d_nchw16c_host(torch.from_numpy(x).pin_memory(), pw, torch.from_numpy(b).cuda(),
                                  stride=layer.stride, pad=layer.pad, relu=True, chunk=1)
        torch.cuda.synchronize()
        y = y.numpy()
    else:
        y = P.conv2d_nchw16c(torch.from_numpy(x).cuda(), pw, torch.from_numpy(b).cuda(), stride=layer.stride,
                             pad=layer.pad, relu=True, cfg=cfg).cpu().numpy()
    ref = oracle.conv2d_f64(x, w, b, stride=layer.stride, pad=layer.pad, relu=True)
    return rel(y, ref)


def main(fam):
    assert P.device_ok()
    if fam == "stem":
        err = conv_case(W.ConvLayer(0, 3, 64, 32, 7, 2), 1)
    elif fam == "halo":
        err = conv_case(W.ConvLayer(0, 64, 64, 14, 3, 1), 1)
    elif fam == "resident":
        err = conv_case(W.ConvLayer(0, 64, 256, 14, 1, 1), 1)
    elif fam == "splitk":
        err = conv_case(W.ConvLayer(0, 256, 128, 7, 3, 1), 1, cfg={"split_k": 3})
    elif fam == "host":
        err = conv_case(W.ConvLayer(0, 32, 64, 8, 3, 1), 3, host=True)
    elif fam == "layout":
        x = torch.rand((1, 20, 9, 9), device="cuda")
        back = P.from_nchw16c(P.to_nchw16c(x), 20)
        err = float((back - x).abs().max())
    elif fam in ("gemm", "gemm_splitk", "simt"):
        m, n, k = {"gemm": (256, 128, 96), "gemm_splitk": (128, 64, 1024), "simt": (37, 45, 29)}[fam]
        a, b = W.gemm_inputs(m, n, k, seed=4)
        cfg = {"split_k": 4} if fam == "gemm_splitk" else None
        c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg=cfg,
                   mode="fp32" if fam == "simt" else "3xtf32")
        err = rel(c.cpu().numpy(), oracle.gemm_f64(a, b))
    else:
        raise SystemExit(f"unknown family {fam}")
    torch.cuda.synchronize()
    print(f"{fam}: max-rel {err:.2e}")
    sys.exit(0 if err <= 1e-5 else 1)


if __name__ == "__main__":
    main(sys.argv[1])
