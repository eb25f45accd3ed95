import os, sys, subprocess
if len(sys.argv) == 1:
    for v in range(2):
        env = dict(os.environ, PDL_DEBUG_GEMM=str(v))
        print("=== variant", v, flush=True)
        subprocess.run([sys.executable, __file__, "x"], env=env)
    sys.exit(0)
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
for (M, N, K) in [(128, 64, 32), (256, 128, 96)]:
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32); b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode="tf32"); torch.cuda.synchronize()
    ref = a.astype(np.float64) @ b
    print(M, N, K, "rel", np.abs(c.cpu().numpy() - ref).max() / np.abs(ref).max(), flush=True)
