import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2006_02230_b200 as P
np.set_printoptions(linewidth=200, precision=3, suppress=True)
M, N, K = 128, 64, 32
rng = np.random.default_rng(0)
cases = {
  "A=1,B=1": (np.ones((M, K)), np.ones((K, N))),
  "A=1,B=rand": (np.ones((M, K)), rng.uniform(-1,1,(K,N))),
  "A=rand,B=1": (rng.uniform(-1,1,(M,K)), np.ones((K,N))),
  "A=eye,B=ar": (np.eye(M, K), np.arange(K*N).reshape(K,N)/100.0),
}
for name, (a, b) in cases.items():
    a = a.astype(np.float32); b = b.astype(np.float32)
    c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode="tf32").cpu().numpy()
    ref = a.astype(np.float64) @ b.astype(np.float64)
    print(name, "maxerr", np.abs(c-ref).max(), "max|c|", np.abs(c).max())
    print(" c[0:3,0:10]=", c[0:3,0:10]); print(" r[0:3,0:10]=", ref[0:3,0:10])
    nz = np.argwhere(np.abs(c) > 0)
    print(" nonzero count", len(nz), nz[:5].tolist())
