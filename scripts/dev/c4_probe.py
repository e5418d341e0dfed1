"""Dev: acceptance C4's shape (b=100, c=10, 256 blocks, energy 0.98, L=8000):
wall time of a stitched query (answer to the host) vs naive_range_svd."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1805_00754_b200 as z
rng = np.random.default_rng(1004)
b, c, nb = 100, 10, 256
lat = np.cumsum(rng.standard_normal((b * nb, 2)) * 0.4, axis=0) * 0.05
raw = lat @ rng.standard_normal((2, c)) + 0.01 * rng.standard_normal((b * nb, c))
st = z.BlockStore(b, c, 0.98)
st.append(raw)
snap = st.snapshot()
L = 8000
offs = rng.integers(0, b * nb - L, 9)
for rep in range(2):
    fast, naive = [], []
    for t0 in offs:
        t0 = int(t0)
        h = time.perf_counter(); z.range_query(snap, t0, t0 + L - 1, z.Truncation.energy(0.98)); fast.append(time.perf_counter() - h)
        h = time.perf_counter(); z.naive_range_svd(snap, t0, t0 + L - 1); naive.append(time.perf_counter() - h)
    print("fast median ms %.3f  naive median ms %.3f" % (1e3 * np.median(fast), 1e3 * np.median(naive)), flush=True)
