"""One cfg2 similar_range_search call (20,000-row windows, stride 500). Dev tool."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
raw = workloads.generate("cfg2")
st = z.BlockStore(2000, 64, policy=z.Truncation.fixed_rank(20))
st.append(raw)
snap = st.snapshot()
bf = raw.shape[0] - 20000
for i in range(2):
    t0 = time.perf_counter()
    hits = z.similar_range_search(snap, bf, bf + 19999, 500, 10)
    print("search", round(time.perf_counter() - t0, 4), "s", hits[0], flush=True)
