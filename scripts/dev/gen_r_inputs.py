"""Dev: R factors (64 x 64, upper triangular, row-major) of cfg2 blocks and of
cfg2 query stitch stacks, for scripts/dev/m2_variants.cu."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1805_00754_b200 import workloads
raw = workloads.generate("cfg2", rows=400 * 2000)
Rs = []
for i in range(240):
    Rs.append(np.linalg.qr(raw[i * 2000:(i + 1) * 2000], mode="r"))
# stitch stacks: rank-20 block factors, 160 consecutive blocks -> 3200 x 64
facs = []
for i in range(400):
    u, s, vt = np.linalg.svd(raw[i * 2000:(i + 1) * 2000], full_matrices=False)
    facs.append(s[:20, None] * vt[:20])
for j in range(16):
    st = np.vstack(facs[j * 15: j * 15 + 160])
    Rs.append(np.linalg.qr(st, mode="r"))
R = np.stack(Rs).astype(np.float64)
R.tofile("/tmp/r_inputs.bin")
np.stack([np.linalg.svd(r, compute_uv=False) for r in R]).astype(np.float64).tofile("/tmp/r_inputs_sv.bin")
print(R.shape)
