"""Break down the storage e2e (host rows -> append -> spectrum): pinned H2D
bandwidth, host scan cost, append wall time. Dev tool, not part of the bench."""
import ctypes as C
import time

import numpy as np
import torch

import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads

L = _capi.lib()
cfg = workloads.CONFIGS["cfg2"]
raw = workloads.generate("cfg2")
nbytes = raw.nbytes
h = C.c_void_p()
assert L.zsvd_host_alloc(nbytes, C.byref(h)) == 0
C.memmove(h, raw.ctypes.data, nbytes)
hp = np.ctypeslib.as_array((C.c_double * raw.size).from_address(h.value)).reshape(raw.shape)
d = torch.empty(raw.size, dtype=torch.float64, device="cuda")
for _ in range(3):
    assert L.zsvd_memcpy(C.c_void_p(d.data_ptr()), h, nbytes, None) == 0
    L.zsvd_stream_sync(None)
t = []
for _ in range(5):
    t0 = time.perf_counter()
    L.zsvd_memcpy(C.c_void_p(d.data_ptr()), h, nbytes, None)
    L.zsvd_stream_sync(None)
    t.append(time.perf_counter() - t0)
print(f"pinned H2D 512MB: {min(t)*1e3:.2f} ms = {nbytes/min(t)/1e9:.1f} GB/s")
t0 = time.perf_counter()
np.isfinite(hp).all()
print(f"numpy isfinite scan: {(time.perf_counter()-t0)*1e3:.2f} ms")
st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
nb = raw.shape[0] // cfg.b
sig = np.zeros((nb, cfg.k)); rk = np.zeros(nb, dtype=np.uint32)
for i in range(6):
    L.zsvd_store_reset(st._h)
    t0 = time.perf_counter()
    assert L.zsvd_store_append(st._h, h, raw.shape[0], cfg.c, _capi.MEM_HOST) == 0
    t1 = time.perf_counter()
    L.zsvd_store_sync(st._h)
    t2 = time.perf_counter()
    L.zsvd_store_spectrum(st._h, 0, nb, sig.ctypes.data, cfg.k, rk.ctypes.data)
    t3 = time.perf_counter()
    print(f"append host: enqueue+scan {1e3*(t1-t0):.2f} ms, drain {1e3*(t2-t1):.2f} ms, spectrum {1e3*(t3-t2):.2f} ms, total {1e3*(t3-t0):.2f}")
dd = C.c_void_p(d.data_ptr())
for i in range(3):
    L.zsvd_store_reset(st._h)
    t0 = time.perf_counter()
    assert L.zsvd_store_append(st._h, dd, raw.shape[0], cfg.c, _capi.MEM_DEVICE) == 0
    L.zsvd_store_sync(st._h)
    print(f"append device: {1e3*(time.perf_counter()-t0):.2f} ms")
