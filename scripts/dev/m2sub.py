import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
raw = workloads.generate("cfg2", rows=4000)
for i in range(3):
    z.thin_svd(raw[:2000])
st = np.random.default_rng(0).standard_normal((3200, 64)) * np.logspace(0, -3, 64)
for i in range(3):
    z.thin_svd(st)
