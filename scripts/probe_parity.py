import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle
import paper_2006_02230_b200 as P
torch.manual_seed(0)
def rel(a, b): return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
ok = True
for mode, tol in (("3xtf32", 1e-5), ("tf32", 1e-2), ("fp32", 1e-5)):
    for (m, n, k) in [(128, 128, 32), (256, 256, 256), (300, 192, 100), (1024, 1024, 1024), (49, 2048, 512), (3136, 64, 576), (37, 45, 29)]:
        rng = np.random.default_rng(1)
        a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        c = P.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode=mode).cpu().numpy()
        r = rel(c, oracle.gemm_f64(a, b))
        print(f"gemm {mode} {m}x{n}x{k}: rel={r:.3e}", "OK" if r <= tol else "FAIL", flush=True)
        ok &= r <= tol
import glob
for path in sorted(glob.glob('tests/golden/conv_*.npz')):
    g = np.load(path)
    bias = torch.from_numpy(g['bias']).cuda() if 'bias' in g.files else None
    for mode, tol in (("3xtf32", 1e-5), ("tf32", 1e-2), ("fp32", 1e-5)):
        y = P.conv2d_nchw16c(torch.from_numpy(g['x']).cuda(), torch.from_numpy(g['w']).cuda(), bias, stride=int(g['stride']), pad=int(g['pad']), relu=bool(g['relu']), mode=mode).cpu().numpy()
        r = rel(y, g['y'])
        print(f"{path.split('/')[-1]} {mode}: rel={r:.3e}", "OK" if r <= tol else "FAIL", flush=True)
        ok &= r <= tol
print("ALL_OK" if ok else "SOME_FAIL")
