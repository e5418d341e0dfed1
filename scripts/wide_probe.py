"""Device-input storage of N blocks of cfg3 / cfg5 (wide path), timed with
CUDA events on the store stream. Dev tool: python scripts/wide_probe.py cfg3 64"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
name, nb = sys.argv[1], int(sys.argv[2])
cfg = workloads.CONFIGS[name]
L = _capi.lib()
t0 = time.time()
raw = workloads.generate(name, rows=nb * cfg.b)
print("generated", raw.shape, f"{time.time() - t0:.1f}s", flush=True)
ptr = C.c_void_p()
assert L.zsvd_device_alloc(raw.nbytes, 0, C.byref(ptr)) == 0
assert L.zsvd_memcpy(ptr, raw.ctypes.data, raw.nbytes, None) == 0
L.zsvd_stream_sync(None)
st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
stream = C.c_void_p(st.stream())
e0, e1 = C.c_void_p(), C.c_void_p()
L.zsvd_event_create(C.byref(e0)); L.zsvd_event_create(C.byref(e1))
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    L.zsvd_store_reset(st._h)
    L.zsvd_event_record(e0, stream)
    rc = L.zsvd_store_append(st._h, ptr, raw.shape[0], cfg.c, _capi.MEM_DEVICE)
    L.zsvd_event_record(e1, stream)
    L.zsvd_store_sync(st._h)
    ms = C.c_float(); L.zsvd_event_elapsed_ms(e0, e1, C.byref(ms))
    print(name, nb, "blocks: rc", rc, f"{ms.value:.1f} ms = {ms.value / nb:.3f} ms/block, {raw.shape[0] / ms.value * 1e3:.3e} rows/s", flush=True)
f = st.block(0)
print("block0 rank", f.rank(), "sigma[:3]", f.sigma[:3], "defect", np.abs(f.u.T @ f.u - np.eye(f.rank())).max())
