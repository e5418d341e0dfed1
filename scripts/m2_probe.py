"""Phase times (ZSVD_PHASE_TIMES=1) and M2 sub-phase clocks (ZSVD_DEBUG=1):
single-task thin_svd, then device-input storage flushes of 500 / 64 / 8
blocks. Dev tool."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
L = _capi.lib()
raw = workloads.generate("cfg2")
for rep in range(2):
    z.thin_svd(raw[:2000])
ptr = C.c_void_p()
assert L.zsvd_device_alloc(raw.nbytes, 0, C.byref(ptr)) == 0
assert L.zsvd_memcpy(ptr, raw.ctypes.data, raw.nbytes, None) == 0
L.zsvd_stream_sync(None)
for nb in (500, 500, 148, 296, 444, 64, 8):
    st = z.BlockStore(2000, 64, policy=z.Truncation.fixed_rank(20))
    st.append_ptr(ptr.value, nb * 2000, 64, _capi.MEM_DEVICE)
    st.block(0)
print("fallbacks", z.fallback_count())
