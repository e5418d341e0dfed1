"""Parity on every BASELINE.json config at its own shape.

The GPU answers are compared with the oracle restatement of the reference
(oracle/zsvd_oracle.c, DIRECT block mode with the LAPACK backend, justified by
store_test.cpp:112-121 / acceptance C6 and checked against the row-by-row
INCREMENTAL mode in test_gpu_baseline_parity.py) computed from the SAME raw
rows, end to end: raw rows -> oracle block factors -> oracle range_query
(query.hpp:163-191) on one side, raw rows -> GPU store -> GPU range_query on
the other.  Tolerances are north_star's (tests/parity.py).

  cfg2  all 500 blocks, three L = 3.2e5 queries (161-block stitches)
  cfg3  100 blocks (4000 x 256), two L = 3.2e5 queries (81-block wide stitches)
  cfg4  2e5 rows ingested in 100-row chunks, a query every 10,000 rows
  cfg5  20 blocks (8192 x 1024) + a 1,152-row open tail: two blocks, a
        17-block wide stitch (K = 1088 >= c = 1024 stacked rows) and a range
        ending in the open tail
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
from parity import assert_parity, defect

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, min(32, os.cpu_count() or 1))


def fixed(k):
    return z.Truncation.fixed_rank(k)


def oracle_blocks(raw, b, k, idxs, open_tail=False):
    """Oracle DIRECT factors (store.hpp:234-240 seal: SVD -> truncate -> sign) of
    the given sealed blocks, computed in a thread pool (one oracle store per
    block); with open_tail, also the open block (untruncated, store.hpp:59-62)."""
    O.set_backend("lapack")

    def one(i):
        st = O.Store(b, raw.shape[1], 1.0, policy=O.FIXED_RANK, k=k, mode=O.DIRECT)
        st.append(raw[i * b:(i + 1) * b])
        return i, st.block(0)

    with ThreadPoolExecutor(THREADS) as ex:
        out = dict(ex.map(one, sorted(set(idxs))))
    if open_tail:
        nb = raw.shape[0] // b
        st = O.Store(b, raw.shape[1], 1.0, policy=O.FIXED_RANK, k=k, mode=O.DIRECT)
        st.append(raw[nb * b:])
        out[nb] = st.block(0)
    return out


def oracle_query(blocks, b, first, last, k):
    """range_query (query.hpp:163-191) with oracle primitives on oracle blocks."""
    S, E = first // b, last // b
    if S == E:
        f = O.trim_block(blocks[S], first - S * b, last - S * b, O.FIXED_RANK, 1.0, k)
    else:
        head = O.trim_block(blocks[S], first - S * b, b - 1, O.FIXED_RANK, 1.0, k)
        tail = O.trim_block(blocks[E], 0, last - E * b, O.FIXED_RANK, 1.0, k)
        f = O.stitch([head] + [blocks[i] for i in range(S + 1, E)] + [tail], O.FIXED_RANK, 1.0, k)
    return O.canonical_sign(f)


def check_query(snap, blocks, b, first, last, k, what):
    ans = z.range_query(snap, first, last, fixed(k)).factors
    assert ans.left_rows() == last - first + 1
    assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8
    return assert_parity(ans, oracle_query(blocks, b, first, last, k), what=what)


def test_cfg2_full_end_to_end():
    """cfg2 at its BASELINE size: 1e6 x 64 rows into the GPU store (500 blocks);
    every block of three L = 3.2e5 ranges against the oracle's DIRECT blocks, and
    the queries against the oracle's query on its own blocks."""
    cfg = workloads.CONFIGS["cfg2"]
    raw = workloads.generate("cfg2")
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    g.append(raw)
    assert g.sealed_count() == 500
    L = 320_000
    offs = [int(t) for t in workloads.query_offsets(cfg.t, L, 3, seed=42)]
    need = set()
    for t0 in offs:
        need.update(range(t0 // cfg.b, (t0 + L - 1) // cfg.b + 1))
    blocks = oracle_blocks(raw, cfg.b, cfg.k, need)
    worst = [0.0, 0.0, 0.0]
    for i in sorted(need):
        e = assert_parity(g.block(i), blocks[i], what=f"cfg2 block {i}")
        worst = [max(a, w) for a, w in zip(e, worst)]
    print("cfg2 blocks worst (sigma, recon, angle):", worst, "over", len(need), "blocks")
    snap = g.snapshot()
    for t0 in offs:
        e = check_query(snap, blocks, cfg.b, t0, t0 + L - 1, cfg.k, f"cfg2 L=3.2e5 at {t0}")
        print("cfg2 query", t0, e)


def test_cfg3_long_queries():
    """cfg3 (4000 x 256, k = 30): 100 blocks; L = 3.2e5 queries span 81-82
    blocks, i.e. a 2,430-row x 256 wide stitch."""
    cfg = workloads.CONFIGS["cfg3"]
    nb = 100
    raw = workloads.generate("cfg3", rows=nb * cfg.b)
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    g.append(raw)
    L = 320_000
    offs = [int(t) for t in workloads.query_offsets(nb * cfg.b, L, 2, seed=42)]
    need = set()
    for t0 in offs:
        need.update(range(t0 // cfg.b, (t0 + L - 1) // cfg.b + 1))
    blocks = oracle_blocks(raw, cfg.b, cfg.k, need)
    for i in sorted(need)[::10]:
        assert_parity(g.block(i), blocks[i], what=f"cfg3 block {i}")
    snap = g.snapshot()
    for t0 in offs:
        e = check_query(snap, blocks, cfg.b, t0, t0 + L - 1, cfg.k, f"cfg3 L=3.2e5 at {t0}")
        print("cfg3 query", t0, e)


def test_cfg4_streaming_ingest():
    """cfg4 (1000 x 32, k = 10): rows arrive in 100-row chunks, a block's SVD
    fires on fill, one query (L ~ U[1e4, 3.2e5] clamped to total_rows) after
    every 10,000 ingested rows (BASELINE configs[3])."""
    cfg = workloads.CONFIGS["cfg4"]
    rows = 200_000
    raw = workloads.generate("cfg4", rows=rows)
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    blocks = oracle_blocks(raw, cfg.b, cfg.k, range(rows // cfg.b))
    rng = np.random.default_rng(44)
    nq = 0
    for i in range(0, rows, 100):
        g.append(raw[i:i + 100])
        total = i + 100
        if total % 10_000 == 0:
            L = min(int(rng.integers(10_000, 320_001)), total)
            t0 = int(rng.integers(0, total - L + 1))
            check_query(g.snapshot(), blocks, cfg.b, t0, t0 + L - 1, cfg.k, f"cfg4 ingest {total} [{t0},+{L}]")
            nq += 1
    assert nq == 20 and g.sealed_count() == rows // cfg.b
    for i in range(0, rows // cfg.b, 17):
        assert_parity(g.block(i), blocks[i], what=f"cfg4 block {i}")
    inc = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.INCREMENTAL)
    inc.append(raw[:2 * cfg.b])
    for i in range(2):
        assert_parity(g.block(i), inc.block(i), what=f"cfg4 block {i} vs row-by-row reference")


def test_cfg5_blocks_and_wide_stitch():
    """cfg5 (8192 x 1024, k = 64): two blocks against the oracle's DIRECT
    (LAPACK) blocks; a 17-block range whose stitch stacks 1,088 >= c = 1,024
    rows; a range ending in the 1,152-row open tail (BASELINE configs[4])."""
    cfg = workloads.CONFIGS["cfg5"]
    nb = 20
    raw = workloads.generate("cfg5", rows=nb * cfg.b + 1152)
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    g.append(raw)
    assert g.sealed_count() == nb and g.open_rows() == 1152
    first = 3 * cfg.b + 2500
    last = first + 16 * cfg.b - 1  # blocks 3 .. 19: 17 parts
    tail_first = nb * cfg.b - 5000
    need = set(range(first // cfg.b, last // cfg.b + 1)) | {0, nb - 1, tail_first // cfg.b}
    blocks = oracle_blocks(raw, cfg.b, cfg.k, need, open_tail=True)
    for i in (0, 7):
        fg = g.block(i)
        assert defect(fg.u) <= 1e-10 and defect(fg.v) <= 1e-10
        assert_parity(fg, blocks[i], what=f"cfg5 block {i}")
    snap = g.snapshot()
    e = check_query(snap, blocks, cfg.b, first, last, cfg.k, "cfg5 17-block stitch")
    print("cfg5 17-block stitch", e)
    e = check_query(snap, blocks, cfg.b, tail_first, raw.shape[0] - 1, cfg.k, "cfg5 range into the open tail")
    print("cfg5 open-tail range", e)
