"""Small, ncu-friendly run of the hot path: one storage launch over `--blocks`
cfg2 blocks, then `--queries` range queries per length.  Prints timings and the
fallback counter (no ncu needed for those)."""
import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1805_00754_b200 as z  # noqa: E402
from paper_1805_00754_b200 import _capi, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=200)
ap.add_argument("--queries", type=int, default=3)
ap.add_argument("--lengths", default="10000")
ap.add_argument("--skip-storage-repeat", action="store_true")
a = ap.parse_args()
cfg = workloads.CONFIGS["cfg2"]
raw = workloads.generate("cfg2", rows=a.blocks * cfg.b)
L = _capi.lib()
d = C.c_void_p()
assert L.zsvd_device_alloc(raw.nbytes, 0, C.byref(d)) == 0
assert L.zsvd_memcpy(d, raw.ctypes.data, raw.nbytes, None) == 0
assert L.zsvd_stream_sync(None) == 0
s = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
s.profile(True)
t0 = time.perf_counter()
s.append_ptr(d.value, raw.shape[0], cfg.c, _capi.MEM_DEVICE)
print("storage wall ms", (time.perf_counter() - t0) * 1e3, "profile", s.profile_read())
print("fallbacks after storage", z.fallback_count())
snap = s.snapshot()
for Lq in [int(x) for x in a.lengths.split(",")]:
    offs = workloads.query_offsets(raw.shape[0], Lq, a.queries, seed=42)
    for t in offs:
        h0 = time.perf_counter()
        f = snap.query_device(int(t), int(t) + Lq - 1, z.Truncation.fixed_rank(cfg.k))
        k = f.rank()
        print(f"query L={Lq} at {int(t)}: rank {k} wall {1e3 * (time.perf_counter() - h0):.3f} ms")
print("fallbacks after queries", z.fallback_count())
