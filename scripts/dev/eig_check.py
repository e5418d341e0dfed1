"""Dev: compares eig_bench outputs with numpy eigh."""
import glob, os
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
for f in sorted(glob.glob(os.path.join(HERE, "eig_data", "*.bin"))):
    out = f.replace(".bin", ".out")
    if not os.path.exists(out):
        continue
    b = open(f, "rb").read(); n = int(np.frombuffer(b[:4], np.int32)[0]); G = np.frombuffer(b[4:], np.float64).reshape(n, n)
    o = open(out, "rb").read(); lam = np.frombuffer(o[4:4 + 8 * n], np.float64); V = np.frombuffer(o[4 + 8 * n:], np.float64).reshape(n, n)
    w, U = np.linalg.eigh(G)
    ordr = np.argsort(-lam); lam_s = lam[ordr]; V_s = V[:, ordr]; w = w[::-1]; U = U[:, ::-1]
    l1 = w[0]
    abs_err = np.max(np.abs(lam_s - w)) / l1
    top = min(20, n)
    rel_top = np.max(np.abs(lam_s[:top] - w[:top]) / np.maximum(w[:top], 1e-300))
    orth = np.max(np.abs(V.T @ V - np.eye(n)))
    resid = np.max(np.abs(G @ V_s - V_s * lam_s)) / l1
    rq = np.einsum("ij,ij->j", V_s, G @ V_s)
    rq_rel = np.max(np.abs(rq[:top] - w[:top]) / np.maximum(w[:top], 1e-300))
    print(f"{os.path.basename(f):16s} n={n:3d} lam abs/l1 {abs_err:.1e} rel top{top} {rel_top:.1e} (RQ {rq_rel:.1e}) orth {orth:.1e} resid/l1 {resid:.1e} spread_top {np.sqrt(w[0]/max(w[top-1],1e-300)):.1e}")
