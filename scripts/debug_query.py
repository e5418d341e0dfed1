import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import oracle as O
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
from parity import recon_rel, sigma_rel, defect
cfg = workloads.CONFIGS["cfg2"]
raw = workloads.generate("cfg2", rows=16 * cfg.b + 777)
g = z.BlockStore(cfg.b, cfg.c, policy=z.Truncation.fixed_rank(cfg.k))
g.append(raw)
r = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.DIRECT)
r.append(raw)
fx = z.Truncation.fixed_rank(cfg.k)
def rep(name, fg, fo):
    print(name, "rank", fg.rank(), fo.rank, "sig", sigma_rel(fg.sigma, fo.s) if fg.rank()==fo.rank else None,
          "recon", recon_rel(fg, fo), "defU", defect(fg.u), "defV", defect(fg.v), flush=True)
b15g, b15o = g.block(15), r.block(15)
rep("block15", b15g, b15o)
og, oo = g.block(16), r.block(16)
rep("open", og, oo)
th = z.trim_block(b15g, 1990, 1999, fx); to = O.trim_block(b15o, 1990, 1999, O.FIXED_RANK, 1.0, cfg.k)
rep("head trim", th, to)
tt = z.trim_block(og, 0, 776, fx); tto = O.trim_block(oo, 0, 776, O.FIXED_RANK, 1.0, cfg.k)
rep("tail trim", tt, tto)
st = z.stitch([th, tt], fx); sto = O.stitch([to, tto], O.FIXED_RANK, 1.0, cfg.k)
rep("stitch", st, sto)
q = z.range_query(g, 31990, 32776, fx).factors; qo = r.range_query(31990, 32776)
rep("query", q, qo)
for (a, b) in ((1990, 1999), (0, 9), (5, 24), (3, 5)):
    w = z.thin_svd(raw[a:b+1, :20].T.copy()); wo = O.thin_svd(raw[a:b+1, :20].T.copy())
    rep(f"thin wide^T {b-a+1}", w, wo)
    w = z.thin_svd(raw[a:b+1, :20].copy()); wo = O.thin_svd(raw[a:b+1, :20].copy())
    rep(f"thin wide {b-a+1}x20", w, wo)
print("fallbacks", z.fallback_count())
