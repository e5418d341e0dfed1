"""Dev: storage flush time vs number of cfg2 blocks (device rows)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
L = _capi.lib()
raw = workloads.generate("cfg2", rows=600 * 2000)
ptr = C.c_void_p()
assert L.zsvd_device_alloc(raw.nbytes, 0, C.byref(ptr)) == 0
assert L.zsvd_memcpy(ptr, raw.ctypes.data, raw.nbytes, None) == 0
L.zsvd_stream_sync(None)
st = z.BlockStore(2000, 64, policy=z.Truncation.fixed_rank(20))
s = C.c_void_p(st.stream())
e0, e1 = C.c_void_p(), C.c_void_p()
L.zsvd_event_create(C.byref(e0)); L.zsvd_event_create(C.byref(e1))
ms = C.c_float()
for nb in [int(a) for a in (sys.argv[1:] or [148, 296, 400, 444, 480, 500, 540, 592])]:
    best = 1e9
    for rep in range(4):
        L.zsvd_store_reset(st._h)
        L.zsvd_event_record(e0, s)
        assert L.zsvd_store_append(st._h, ptr, nb * 2000, 64, _capi.MEM_DEVICE) == 0
        L.zsvd_event_record(e1, s)
        L.zsvd_store_sync(st._h)
        L.zsvd_event_elapsed_ms(e0, e1, C.byref(ms))
        if rep: best = min(best, ms.value)
    print(f"blocks {nb:4d}: {best:.3f} ms  {best / nb * 1e3:.2f} us/block", flush=True)
