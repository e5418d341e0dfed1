"""Dev: time pageable cfg2 appends on one reused store (bounce ring)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads, _capi
cfg = workloads.CONFIGS["cfg2"]
raw = workloads.generate("cfg2")
L = _capi.lib()
st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
for rep in range(4):
    L.zsvd_store_reset(st._h)
    t0 = time.perf_counter()
    st.append(raw)
    L.zsvd_store_sync(st._h)
    print("rep", rep, "ms", 1e3 * (time.perf_counter() - t0), flush=True)
