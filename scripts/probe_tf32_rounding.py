"""Does the tcgen05 kind::tf32 datapath truncate or round fp32 operands?
A = 1 + 2^-11 + 2^-12 (0.75 tf32-ulp above 1), B = 1, K = 8: C/8 = tf32(a)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
a_val = np.float32(1 + 2.0**-11 + 2.0**-12)
a = np.zeros((128, 32), np.float32); a[:, :8] = a_val
b = np.zeros((32, 64), np.float32); b[:8, :] = 1
c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode="tf32").cpu().numpy()
v = c[0, 0] / 8
print("tf32(a) as used by the tensor core:", repr(v), "| truncation would give 1.0, RN 1.0009765625")
print("TC_TF32_CONVERSION=" + ("truncate" if v == 1.0 else "round" if v == np.float32(1 + 2**-10) else "other"))
