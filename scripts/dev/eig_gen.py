"""Dev: Gram matrices for the eig harness (scripts/dev/eig_bench.cu): stitch
Grams of cfg1/cfg2/cfg4 queries (oracle block factors) and synthetic cases."""
import os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_1805_00754_b200 import workloads
import oracle as O
O.set_backend("lapack")
D = os.path.join(HERE, "eig_data")
os.makedirs(D, exist_ok=True)

def put(name, G):
    G = np.ascontiguousarray((G + G.T) / 2)
    with open(os.path.join(D, name + ".bin"), "wb") as f:
        f.write(np.int32(G.shape[0]).tobytes()); f.write(G.tobytes())

def stitch_gram(cfg_name, nblocks):
    cfg = workloads.CONFIGS[cfg_name]
    raw = workloads.generate(cfg_name, rows=(nblocks + 2) * cfg.b)
    st = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.DIRECT); st.append(raw)
    S = np.vstack([st.block(i).s[:, None] * st.block(i).v.T for i in range(1, nblocks + 1)])
    return S.T @ S

put("cfg2_161", stitch_gram("cfg2", 161))
put("cfg1_20", stitch_gram("cfg1", 20))
put("cfg4_100", stitch_gram("cfg4", 100))
rng = np.random.default_rng(0)
for n in (16, 32, 64):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    put(f"rand{n}_k1e6", (Q * np.logspace(0, -6, n)) @ Q.T)
    put(f"randgauss{n}", (lambda A: A.T @ A)(rng.standard_normal((3 * n, n))))
put("ident64", np.eye(64))
put("rankdef64", (lambda A: A.T @ A)(rng.standard_normal((20, 64))))
put("diag64", np.diag(rng.uniform(1, 2, 64)))
put("odd37", (lambda A: A.T @ A)(rng.standard_normal((100, 37))))
# near-degenerate pairs (sinusoid-like spectra) and exact ties
n = 64
Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
lamp = np.repeat(np.logspace(0, -5, 32), 2) * (1 + np.tile([0, -1e-9], 32))
put("pairs64", (Q * lamp) @ Q.T)
lamt = np.logspace(0, -5, 64); lamt[3] = lamt[2]
put("tie64", (Q * lamt) @ Q.T)
put("cfg2_3", stitch_gram("cfg2", 3))
print(sorted(os.listdir(D)))
