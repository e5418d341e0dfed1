"""Device-input storage of cfg2 (500 blocks) timed by CUDA events on the store
stream, for the lane count in ZSVD_DEV_LANES. Dev tool."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
L = _capi.lib()
raw = workloads.generate("cfg2")
ptr = C.c_void_p()
assert L.zsvd_device_alloc(raw.nbytes, 0, C.byref(ptr)) == 0
assert L.zsvd_memcpy(ptr, raw.ctypes.data, raw.nbytes, None) == 0
L.zsvd_stream_sync(None)
st = z.BlockStore(2000, 64, policy=z.Truncation.fixed_rank(20))
stream = C.c_void_p(st.stream())
e0, e1 = C.c_void_p(), C.c_void_p()
L.zsvd_event_create(C.byref(e0)); L.zsvd_event_create(C.byref(e1))
ts = []
for i in range(8):
    L.zsvd_store_reset(st._h)
    L.zsvd_event_record(e0, stream)
    assert L.zsvd_store_append(st._h, ptr, raw.shape[0], 64, _capi.MEM_DEVICE) == 0
    L.zsvd_event_record(e1, stream)
    L.zsvd_store_sync(st._h)
    ms = C.c_float(); L.zsvd_event_elapsed_ms(e0, e1, C.byref(ms)); ts.append(ms.value)
print("lanes", os.environ.get("ZSVD_DEV_LANES", "1"), "ms", " ".join(f"{t:.3f}" for t in ts[2:]), "fallbacks", z.fallback_count())
