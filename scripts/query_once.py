"""cfg2 store (device rows) then 5 queries at L = 3.2e5 (for ncu launch lists). Dev tool."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
L = _capi.lib()
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = workloads.CONFIGS[name]
nb = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.t // cfg.b
Lq = int(sys.argv[3]) if len(sys.argv) > 3 else 320_000
raw = workloads.generate(name, rows=nb * cfg.b)
ptr = C.c_void_p()
assert L.zsvd_device_alloc(raw.nbytes, 0, C.byref(ptr)) == 0
assert L.zsvd_memcpy(ptr, raw.ctypes.data, raw.nbytes, None) == 0
L.zsvd_stream_sync(None)
st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
assert L.zsvd_store_append(st._h, ptr, raw.shape[0], cfg.c, _capi.MEM_DEVICE) == 0
snap = st.snapshot()
Lq = min(Lq, raw.shape[0])
offs = workloads.query_offsets(raw.shape[0], Lq, 5, seed=42)
for t0 in offs:
    t0 = int(t0)
    w0 = time.perf_counter()
    res = snap.query_device(t0, t0 + Lq - 1, z.Truncation.fixed_rank(cfg.k))
    L.zsvd_stream_sync(C.c_void_p(snap.stream()))
    print(f"query {t0} wall {1e3 * (time.perf_counter() - w0):.3f} ms", flush=True)
    del res
