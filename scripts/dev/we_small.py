"""Dev: the 300 x 100 k=12 wide store + queries of tests/test_gpu_wide.py, one step per line (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1805_00754_b200 as z
b, c, k = 300, 100, 12
rng = np.random.default_rng(b + c)
t = 5 * b + 77
base = np.sin(np.arange(t)[:, None] / rng.uniform(20, 400, 8)[None, :]) @ rng.standard_normal((8, c))
raw = base + 0.05 * rng.standard_normal((t, c))
g = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
g.append(raw)
print("appended", flush=True)
snap = g.snapshot()
for a0, a1 in [(5, b - 3), (b - 10, b + 20), (17, 3 * b + 5), (0, t - 1), (2 * b + 1, t - 1)]:
    f = z.range_query(snap, a0, a1, z.Truncation.fixed_rank(k)).factors
    print("query", a0, a1, "rank", f.rank(), flush=True)
