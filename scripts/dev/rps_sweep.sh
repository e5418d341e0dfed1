for r in 0 64 128 256 512; do
  echo "== uform rows $r"; ZSVD_UFORM_ROWS=$r ZSVD_PHASE_TIMES=1 python scripts/query_once.py cfg2 500 320000 2>&1 | grep -A0 "ns=.* qf=64" | tail -2
  ZSVD_UFORM_ROWS=$r python - <<'PY'
import ctypes as C, os, sys, statistics
sys.path.insert(0, os.getcwd())
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
L = _capi.lib()
cfg = workloads.CONFIGS["cfg2"]
raw = workloads.generate("cfg2")
st = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k)); st.append(raw)
snap = st.snapshot(); qs = C.c_void_p(snap.stream())
e0, e1 = C.c_void_p(), C.c_void_p(); L.zsvd_event_create(C.byref(e0)); L.zsvd_event_create(C.byref(e1))
ms = C.c_float(); out = []
for t0 in workloads.query_offsets(raw.shape[0], 320000, 40, seed=42):
    t0 = int(t0); L.zsvd_event_record(e0, qs)
    r = snap.query_device(t0, t0 + 319999, z.Truncation.fixed_rank(cfg.k)); L.zsvd_event_record(e1, qs)
    L.zsvd_event_elapsed_ms(e0, e1, C.byref(ms)); out.append(ms.value); del r
print("p50 ms", statistics.median(out[5:]))
PY
done
