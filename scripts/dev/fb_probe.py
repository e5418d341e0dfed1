"""Fallback count and worst U / V defect over the cfg1/cfg2/cfg4 stores (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
for name, rows in (("cfg1", None), ("cfg2", None), ("cfg4", 1_000_000)):
    cfg = workloads.CONFIGS[name]
    raw = workloads.generate(name, rows=rows)
    f0 = z.fallback_count()
    st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
    st.append(raw)
    nb = st.sealed_count()
    du = dv = 0.0
    for i in range(0, nb, max(1, nb // 50)):
        f = st.block(i)
        du = max(du, np.abs(f.u.T @ f.u - np.eye(f.u.shape[1])).max())
        dv = max(dv, np.abs(f.v.T @ f.v - np.eye(f.v.shape[1])).max())
    snap = st.snapshot()
    dq = 0.0
    for t0 in workloads.query_offsets(raw.shape[0], min(320_000, raw.shape[0] // 2), 10, seed=3):
        L = min(320_000, raw.shape[0] // 2)
        q = z.range_query(snap, int(t0), int(t0) + L - 1, z.Truncation.fixed_rank(cfg.k)).factors
        dq = max(dq, np.abs(q.u.T @ q.u - np.eye(q.u.shape[1])).max())
    print(f"{name}: blocks {nb} fallbacks {z.fallback_count() - f0} max U defect {du:.2e} V defect {dv:.2e} query U defect {dq:.2e}", flush=True)
