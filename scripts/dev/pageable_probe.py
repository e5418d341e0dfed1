"""Dev: pageable vs pinned host appends (bounce ring) — correctness and rate."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
for name, rows in (("cfg1", 100_000), ("cfg2", 1_000_000)):
    cfg = workloads.CONFIGS[name]
    raw = workloads.generate(name, rows=rows)
    a = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
    t0 = time.perf_counter(); a.append(raw); a.sync() if hasattr(a, "sync") else None
    print(name, "pageable append ok", time.perf_counter() - t0, flush=True)
    b = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
    for i in range(0, rows, 100):
        b.append(raw[i:i + 100])
    for i in range(0, rows // cfg.b, max(1, rows // cfg.b // 7)):
        fa, fb = a.block(i), b.block(i)
        assert np.array_equal(fa.u, fb.u) and np.array_equal(fa.sigma, fb.sigma), i
    print(name, "bitwise vs 100-row appends ok", flush=True)
    for rep in range(3):
        a2 = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
        t0 = time.perf_counter(); a2.append(raw); a2.block(0)
        print(name, "pageable append s", time.perf_counter() - t0, flush=True)
