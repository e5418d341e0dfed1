"""Times single thin_svd calls of several shapes (ZSVD_DEBUG=1 prints sweeps)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
rng = np.random.default_rng(0)
cases = [rng.standard_normal((64, 64)), rng.standard_normal((2000, 64)), rng.standard_normal((120, 64)),
         rng.standard_normal((2000, 20)), workloads.generate("cfg2", rows=2000), rng.standard_normal((16, 16))]
for a in cases:
    for rep in range(2):
        t0 = time.perf_counter()
        f = z.thin_svd(a)
        print(a.shape, "rank", f.rank(), "ms", round((time.perf_counter() - t0) * 1e3, 3), flush=True)
print("fallbacks", z.fallback_count())
