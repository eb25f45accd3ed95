"""B200-native (sm_100a) implementation of the PolyDL (arXiv 2006.02230) hot path:
fp32 blocked convolution (nChw16c / KCRS16c16k), row-major fp32 GEMM and the
fused conv + bias + ReLU operator, behind the reference `looprank` package's
loop-nest entry points (see loopdsl.py / executor.py) and ranking API.

Kernels live in libpdl.so (csrc/, C ABI in include/pdl.h); there is no CPU
fallback on this path.
"""
from ._lib import PdlDeviceError, PdlError, PdlShapeError, TileCfg  # noqa: F401
from . import ops  # noqa: F401
from .ops import (PackedWeights, SimtPathWarning, accumulate_, bias_relu_, conv2d_nchw,  # noqa: F401
                  conv2d_nchw16c, conv2d_nchw16c_host, conv_out_hw,
                  device_ok, from_nchw16c, gemm, prepack_weights, to_nchw16c, to_nchw4c,
                  weights_to_kcrs16c16k)

from .loopnest import (LoopDslError, LoopNest, NonAffineError, ParseError, Program,  # noqa: F401
                       parse, parse_program, pretty, reinstate_microkernel,
                       substitute_microkernel)
from .executor import InterpreterError, execute, interpret, make_inputs, plan_program  # noqa: F401
from .fusion import (FusedNest, FusionDecision, FusionError, OperatorPair, can_fuse,  # noqa: F401
                     fuse, write_set)

__version__ = "0.1.0"
