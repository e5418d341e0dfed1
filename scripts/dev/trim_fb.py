"""Fallback counter around single cfg2 queries (fused trims debugging). Dev tool."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
L = _capi.lib()
cfg = workloads.CONFIGS["cfg2"]
raw = workloads.generate("cfg2", rows=200 * cfg.b)
st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
st.append(raw)
snap = st.snapshot()
for t0 in (450, 1000, 1999, 12345, 60690 % 300000):
    f0 = z.fallback_count()
    res = snap.query_device(t0, t0 + 320000 - 1 if t0 + 320000 <= raw.shape[0] else raw.shape[0] - 1, z.Truncation.fixed_rank(cfg.k))
    L.zsvd_stream_sync(C.c_void_p(snap.stream()))
    print("t0", t0, "fallbacks during query", z.fallback_count() - f0, flush=True)
