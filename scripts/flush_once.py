"""One cfg2 storage flush of 500 device-resident blocks (for ncu launch lists). Dev tool."""
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
assert L.zsvd_store_append(st._h, ptr, raw.shape[0], 64, _capi.MEM_DEVICE) == 0
L.zsvd_store_sync(st._h)
print("ok", z.fallback_count())
