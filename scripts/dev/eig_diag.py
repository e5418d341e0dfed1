"""Dev: where does a cfg4 query's error come from?  Per-block parity of the GPU
store against oracle DIRECT blocks, then the same query on the GPU store and on
a GPU store rebuilt from the oracle's block factors (from_parts)."""
import os, sys, ctypes as C
HERE = os.path.dirname(os.path.abspath(__file__)); ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import oracle as O
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads, _capi
from parity import sigma_rel, recon_rel, max_angle, _uv
from test_gpu_configs_parity import oracle_blocks, oracle_query
cfg = workloads.CONFIGS["cfg4"]
nb = 150
raw = workloads.generate("cfg4", rows=nb * cfg.b)
g = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k)); g.append(raw)
blocks = oracle_blocks(raw, cfg.b, cfg.k, range(nb))
worst = (0, 0, 0)
for i in range(nb):
    fg = g.block(i); fr = blocks[i]
    e = (sigma_rel(_uv(fg)[1], _uv(fr)[1]), recon_rel(fg, fr), i)
    s = np.linalg.svd(raw[i*cfg.b:(i+1)*cfg.b], compute_uv=False)
    if e[1] > worst[1]: worst = (e[0], e[1], i, s[0], s[cfg.k-1], s[cfg.k])
print("worst block (sigma, recon, idx, s1, sk, sk+1):", worst)
ref = oracle_query(blocks, cfg.b, 0, nb * cfg.b - 1, cfg.k)
ans = z.range_query(g, 0, nb * cfg.b - 1, z.Truncation.fixed_rank(cfg.k)).factors
print("query on GPU store: sigma %.2e recon %.2e" % (sigma_rel(_uv(ans)[1], _uv(ref)[1]), recon_rel(ans, ref)))
s = ref.s; print("stitch spectrum top/k/next:", s[0], s[-1])
g2 = z.store_from_parts(cfg.b, cfg.c, z.Truncation.fixed_rank(cfg.k), [blocks[i] for i in range(nb)])
ans2 = z.range_query(g2, 0, nb * cfg.b - 1, z.Truncation.fixed_rank(cfg.k)).factors
print("query on oracle-block store: sigma %.2e recon %.2e" % (sigma_rel(_uv(ans2)[1], _uv(ref)[1]), recon_rel(ans2, ref)))
S = np.vstack([blocks[i].s[:, None] * blocks[i].v.T for i in range(nb)])
sv = np.linalg.svd(S, compute_uv=False)
print("stack sigma 1, k-1, k, k+1, k+2:", sv[0], sv[cfg.k - 2:cfg.k + 2])
print("boundary gap rel sigma1: %.3e" % ((sv[cfg.k - 1] - sv[cfg.k]) / sv[0]))
lam = sv ** 2
print("guard lhs %.3e rhs %.3e" % (4 * 2.22e-16 * lam[0] * sv[cfg.k - 1], 1e-10 * (lam[cfg.k - 1] - lam[cfg.k]) * sv[0]))
# exact answer from the stack: V_exact = right singular vectors of S
_, sv2, vt = np.linalg.svd(S, full_matrices=False)
Vx = vt[:cfg.k].T
Vg = ans2.v
print("V angles (|cos| per column):", np.round(1 - np.abs(np.sum(Vx * Vg, axis=0)), 16))
P = Vx @ Vx.T
print("span error ||(I - PxPx^T) Vg||: %.3e" % np.linalg.norm(Vg - P @ Vg, 2))
Ug = ans2.u
print("U defect %.3e" % np.max(np.abs(Ug.T @ Ug - np.eye(Ug.shape[1]))))
Ar = np.vstack([blocks[i].u @ (blocks[i].s[:, None] * blocks[i].v.T) for i in range(nb)])
rec_g = Ug @ (ans2.sigma[:, None] * Vg.T)
rec_x = Ar @ P
print("recon vs A Vx Vx^T: %.3e ; vs oracle: %.3e" % (np.linalg.norm(rec_g - rec_x) / np.linalg.norm(rec_x), recon_rel(ans2, ref)))
print("A Vg Vg^T vs rec_g: %.3e" % (np.linalg.norm(Ar @ Vg @ Vg.T - rec_g) / np.linalg.norm(rec_x)))
rr = ref.u @ (ref.s[:, None] * ref.v.T)
print("oracle vs A Vx Vx^T: %.3e" % (np.linalg.norm(rr - rec_x) / np.linalg.norm(rec_x)))
