"""Dev: where a cfg2 range query's time goes — event time (as bench.py takes
it), host wall time of the call, and (ZSVD_QPROF=1) the library's host phases.
python scripts/dev/qprof.py [nblocks] [L ...]"""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1805_00754_b200 as z  # noqa: E402
from paper_1805_00754_b200 import _capi, workloads  # noqa: E402


def ck(rc):
    if rc:
        raise RuntimeError(rc)


def main():
    nblocks = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    lengths = [int(x) for x in sys.argv[2:]] or [10000, 320000]
    L = _capi.lib()
    cfg = workloads.CONFIGS["cfg2"]
    rows = nblocks * cfg.b
    raw = workloads.generate("cfg2", rows=rows)
    st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
    st.append(raw)
    snap = st.snapshot()
    qs = C.c_void_p(snap.stream())
    e0, e1 = C.c_void_p(), C.c_void_p()
    ck(L.zsvd_event_create(C.byref(e0)))
    ck(L.zsvd_event_create(C.byref(e1)))
    ms = C.c_float()
    trunc = z.Truncation.fixed_rank(cfg.k)
    for Lq in lengths:
        offs = workloads.query_offsets(rows, Lq, 30, seed=42)
        ev, wall = [], []
        for i in range(33):
            t0 = int(offs[i % 30])
            h0 = time.perf_counter()
            ck(L.zsvd_event_record(e0, qs))
            res = snap.query_device(t0, t0 + Lq - 1, trunc)
            ck(L.zsvd_event_record(e1, qs))
            h1 = time.perf_counter()
            ck(L.zsvd_event_elapsed_ms(e0, e1, C.byref(ms)))
            if i >= 3:
                ev.append(ms.value * 1e3)
                wall.append((h1 - h0) * 1e6)
            del res
        print(f"L={Lq}: event p50 {statistics.median(ev):.1f} us, host wall p50 {statistics.median(wall):.1f} us", flush=True)


if __name__ == "__main__":
    main()
