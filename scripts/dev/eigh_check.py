"""Dev: compares eigh_bench outputs (top-kk eigenpairs) with numpy eigh."""
import glob, os
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
for f in sorted(glob.glob(os.path.join(HERE, "eig_data", "*.bin"))):
    out = f.replace(".bin", ".eigh")
    if not os.path.exists(out):
        continue
    b = open(f, "rb").read(); n = int(np.frombuffer(b[:4], np.int32)[0]); G = np.frombuffer(b[4:], np.float64).reshape(n, n)
    o = open(out, "rb").read(); kk = int(np.frombuffer(o[4:8], np.int32)[0])
    lam = np.frombuffer(o[8:8 + 8 * kk], np.float64); V = np.frombuffer(o[8 + 8 * kk:], np.float64).reshape(n, kk)
    w, U = np.linalg.eigh(G); w = w[::-1]; U = U[:, ::-1]
    l1 = max(w[0], 1e-300)
    abs_err = np.max(np.abs(lam - w[:kk])) / l1
    rel = np.max(np.abs(np.sqrt(np.maximum(lam, 0)) - np.sqrt(np.maximum(w[:kk], 0))) / np.maximum(np.sqrt(np.maximum(w[:kk], 0)), 1e-300))
    orth = np.max(np.abs(V.T @ V - np.eye(kk)))
    resid = np.max(np.abs(G @ V - V * lam)) / l1
    # angle of each vector to the true eigvec where the relative sigma gap > 1e-6
    s = np.sqrt(np.maximum(w, 0)); ang = 0.0
    for j in range(kk):
        gap = min([abs(s[j] - s[i]) for i in (j - 1, j + 1) if 0 <= i < n] + [np.inf]) / max(s[0], 1e-300)
        if gap > 1e-6:
            ang = max(ang, np.sqrt(max(0.0, 1 - min(1.0, abs(U[:, j] @ V[:, j])) ** 2)))
    print(f"{os.path.basename(f):16s} n={n:3d} kk={kk:2d} lam abs/l1 {abs_err:.1e} sigma rel {rel:.1e} orth {orth:.1e} resid/l1 {resid:.1e} angle {ang:.1e} spread {np.sqrt(l1/max(w[kk-1],1e-300)):.1e}")
