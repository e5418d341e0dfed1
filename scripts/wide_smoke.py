import numpy as np, time, sys
sys.path.insert(0, '/root/repo')
import paper_1805_00754_b200 as z
rng = np.random.default_rng(0)
for (m, n) in [(600, 100), (100, 600), (2000, 256), (1500, 1024), (4000, 256)]:
    a = rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -2, n))
    t0 = time.perf_counter()
    f = z.thin_svd(a)
    dt = time.perf_counter() - t0
    s_ref = np.linalg.svd(a, compute_uv=False)
    k = f.rank()
    rel = np.max(np.abs(f.sigma - s_ref[:k]) / s_ref[:k])
    rec = np.linalg.norm((f.u * f.sigma) @ f.v.T - a) / np.linalg.norm(a)
    ou = np.abs(f.u.T @ f.u - np.eye(k)).max(); ov = np.abs(f.v.T @ f.v - np.eye(k)).max()
    print((m, n), "k", k, "sig rel %.2e rec %.2e orthU %.1e orthV %.1e  %.1f ms" % (rel, rec, ou, ov, dt * 1e3), "fallbacks", z.fallback_count(), flush=True)
