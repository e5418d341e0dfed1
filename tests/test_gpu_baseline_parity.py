"""Parity on BASELINE.json's synthetic workloads (north_star bar: sigma and
reconstruction 1e-9 relative, principal angles 1e-7 rad where gaps > 1e-6).

cfg1 (the CPU-runnable oracle case) is checked in full; cfg2 on a block sample
against the oracle, and at its full size (1e6 x 64) through size-independent
properties plus an oracle re-stitch of the GPU's own block factors."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import _capi, workloads
from parity import assert_parity, defect, recon_rel, sigma_rel

pytestmark = pytest.mark.gpu


def fixed(k):
    return z.Truncation.fixed_rank(k)


def oracle_query_from_blocks(blocks, b, first, last, k):
    """range_query (query.hpp:163-191) restated with oracle primitives on given
    block factors (list indexed by block)."""
    S, E = first // b, last // b
    if S == E:
        f = O.trim_block(blocks[S], first - S * b, last - S * b, O.FIXED_RANK, 1.0, k)
    else:
        head = O.trim_block(blocks[S], first - S * b, b - 1, O.FIXED_RANK, 1.0, k)
        tail = O.trim_block(blocks[E], 0, last - E * b, O.FIXED_RANK, 1.0, k)
        f = O.stitch([head] + [blocks[i] for i in range(S + 1, E)] + [tail], O.FIXED_RANK, 1.0, k)
    return O.canonical_sign(f)


def as_oracle(f):
    return O.Factors(np.ascontiguousarray(f.u), np.ascontiguousarray(f.sigma), np.ascontiguousarray(f.v))


@pytest.fixture(scope="module")
def cfg1():
    cfg = workloads.CONFIGS["cfg1"]
    raw = workloads.generate("cfg1")
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    g.append(raw)
    r = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.DIRECT)
    r.append(raw)
    return cfg, raw, g, r


def test_cfg1_storage_all_blocks(cfg1):
    cfg, raw, g, r = cfg1
    assert g.sealed_count() == 100 and g.open_rows() == 0
    worst = [0.0, 0.0, 0.0]
    for i in range(100):
        blk = raw[i * cfg.b:(i + 1) * cfg.b]
        nxt = O.thin_svd(blk).s[cfg.k]
        fg = g.block(i)
        assert defect(fg.u) <= 1e-10 and defect(fg.v) <= 1e-10
        e = assert_parity(fg, r.block(i), sigma_next=nxt, what=f"cfg1 block {i}")
        worst = [max(a, b) for a, b in zip(worst, e)]
    print("cfg1 storage worst (sigma, recon, angle):", worst)


def test_cfg1_storage_vs_incremental_reference(cfg1):
    """The reference's own row-by-row algorithm (store.hpp) on the first blocks."""
    cfg, raw, g, _ = cfg1
    n = 3
    inc = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.INCREMENTAL)
    inc.append(raw[:n * cfg.b])
    for i in range(n):
        nxt = O.thin_svd(raw[i * cfg.b:(i + 1) * cfg.b]).s[cfg.k]
        assert_parity(g.block(i), inc.block(i), sigma_next=nxt, what=f"cfg1 incremental block {i}")


def test_cfg1_queries(cfg1):
    cfg, raw, g, r = cfg1
    rng = np.random.default_rng(11)
    snap = g.snapshot()
    for _ in range(100):
        L = int(rng.integers(10_000, 50_001))
        t0 = int(rng.integers(0, cfg.t - L + 1))
        ans = z.range_query(snap, t0, t0 + L - 1, fixed(cfg.k)).factors
        ref = r.range_query(t0, t0 + L - 1)
        assert ans.left_rows() == L
        assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8
        assert_parity(ans, ref, what=f"cfg1 query [{t0},+{L}]")


def test_cfg1_energy_mode(cfg1):
    """The reference-native energy policy (xi = 0.98) on the same stream."""
    cfg, raw, _, _ = cfg1
    part = raw[:20 * cfg.b + 437]
    g = z.BlockStore(cfg.b, cfg.c, 0.98)
    g.append(part)
    r = O.Store(cfg.b, cfg.c, 0.98, mode=O.DIRECT)
    r.append(part)
    for i in range(20):
        nxt = O.thin_svd(part[i * cfg.b:(i + 1) * cfg.b]).s
        fr = r.block(i)
        assert_parity(g.block(i), fr, sigma_next=nxt[fr.rank] if fr.rank < len(nxt) else 0.0,
                      what=f"energy block {i}")
    snap = g.snapshot()
    for (a, b) in ((0, len(part) - 1), (1234, 15_000), (19_500, len(part) - 1), (3, 950)):
        assert_parity(z.range_query(snap, a, b, 0.98).factors, r.range_query(a, b, 0.98),
                      what=f"energy query [{a},{b}]")


@pytest.fixture(scope="module")
def cfg2_sample():
    cfg = workloads.CONFIGS["cfg2"]
    nb = 16
    raw = workloads.generate("cfg2", rows=nb * cfg.b + 777)
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    g.append(raw)
    r = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.DIRECT)
    r.append(raw)
    return cfg, raw, g, r, nb


def test_cfg2_sample_storage(cfg2_sample):
    cfg, raw, g, r, nb = cfg2_sample
    worst = [0.0, 0.0, 0.0]
    for i in range(nb):
        blk = raw[i * cfg.b:(i + 1) * cfg.b]
        nxt = O.thin_svd(blk).s[cfg.k]
        fg = g.block(i)
        assert defect(fg.u) <= 1e-10 and defect(fg.v) <= 1e-10
        e = assert_parity(fg, r.block(i), sigma_next=nxt, what=f"cfg2 block {i}")
        worst = [max(a, b) for a, b in zip(worst, e)]
    print("cfg2 storage worst (sigma, recon, angle):", worst)
    inc = O.Store(cfg.b, cfg.c, 1.0, policy=O.FIXED_RANK, k=cfg.k, mode=O.INCREMENTAL)
    inc.append(raw[:cfg.b])
    assert_parity(g.block(0), inc.block(0), sigma_next=O.thin_svd(raw[:cfg.b]).s[cfg.k],
                  what="cfg2 block 0 vs row-by-row reference")


def test_cfg2_sample_queries(cfg2_sample):
    cfg, raw, g, r, nb = cfg2_sample
    snap = g.snapshot()
    total = raw.shape[0]
    for L in (10_000, 20_000):
        for t0 in workloads.query_offsets(total, L, 6, seed=42):
            t0 = int(t0)
            ans = z.range_query(snap, t0, t0 + L - 1, fixed(cfg.k)).factors
            assert_parity(ans, r.range_query(t0, t0 + L - 1), what=f"cfg2 query [{t0},+{L}]")
    # open-tail ranges and single-block ranges
    for (a, b) in ((total - 500, total - 1), (nb * cfg.b - 10, total - 1), (4100, 4200), (0, 1999)):
        assert_parity(z.range_query(snap, a, b, fixed(cfg.k)).factors, r.range_query(a, b),
                      what=f"cfg2 [{a},{b}]")


def test_device_input_matches_host_input(cfg2_sample):
    """append from HBM-resident rows == append from host rows, bit for bit."""
    cfg, raw, g, _, nb = cfg2_sample
    L = _capi.lib()
    n = 5 * cfg.b + 123
    part = np.ascontiguousarray(raw[:n])
    ptr = C.c_void_p()
    assert L.zsvd_device_alloc(part.nbytes, 0, C.byref(ptr)) == 0
    try:
        assert L.zsvd_memcpy(ptr, part.ctypes.data, part.nbytes, None) == 0
        assert L.zsvd_stream_sync(None) == 0
        d = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
        d.append_ptr(ptr.value, n, cfg.c, _capi.MEM_DEVICE)
        h = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
        h.append(part)
        for i in range(6):
            a, b = d.block(i), h.block(i)
            assert np.array_equal(a.u, b.u) and np.array_equal(a.sigma, b.sigma) and np.array_equal(a.v, b.v)
        bad = part.copy()
        bad[3 * cfg.b + 7, 5] = np.nan
        assert L.zsvd_memcpy(ptr, bad.ctypes.data, bad.nbytes, None) == 0
        assert L.zsvd_stream_sync(None) == 0
        before = d.total_rows()
        with pytest.raises(z.InvalidInputError):
            d.append_ptr(ptr.value, n, cfg.c, _capi.MEM_DEVICE)
        assert d.total_rows() == before
        # the rejected batch (checked beside the factorisation, then rolled
        # back) left the store as it was: the same rows again agree bit for bit
        assert L.zsvd_memcpy(ptr, part.ctypes.data, part.nbytes, None) == 0
        assert L.zsvd_stream_sync(None) == 0
        d.append_ptr(ptr.value, n, cfg.c, _capi.MEM_DEVICE)
        h.append(part)
        assert d.total_rows() == h.total_rows() == 2 * n
        for i in range(d.sealed_count()):
            a, b = d.block(i), h.block(i)
            assert np.array_equal(a.u, b.u) and np.array_equal(a.sigma, b.sigma) and np.array_equal(a.v, b.v)
        qa = z.range_query(d.snapshot(), 2 * n - 1500, 2 * n - 1, fixed(cfg.k)).factors
        qb = z.range_query(h.snapshot(), 2 * n - 1500, 2 * n - 1, fixed(cfg.k)).factors
        assert np.array_equal(qa.u, qb.u) and np.array_equal(qa.sigma, qb.sigma)
        # a finite entry whose square overflows the block's Gram is not an error:
        # the exact check clears it and the batch stands
        huge = part.copy()
        huge[2 * cfg.b + 5, 3] = 1e200
        assert L.zsvd_memcpy(ptr, huge.ctypes.data, huge.nbytes, None) == 0
        assert L.zsvd_stream_sync(None) == 0
        d2 = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
        d2.append_ptr(ptr.value, n, cfg.c, _capi.MEM_DEVICE)
        assert d2.total_rows() == n
        # NaN in a whole block, in the open block's head and in the tail: rejected
        for where in (2 * cfg.b + 5, 10, n - 3):
            bad = part.copy()
            bad[where, 1] = np.inf if where == 10 else np.nan
            assert L.zsvd_memcpy(ptr, bad.ctypes.data, bad.nbytes, None) == 0
            assert L.zsvd_stream_sync(None) == 0
            before = d2.total_rows()
            with pytest.raises(z.InvalidInputError):
                d2.append_ptr(ptr.value, n, cfg.c, _capi.MEM_DEVICE)
            assert d2.total_rows() == before
    finally:
        L.zsvd_device_free(ptr)


@pytest.mark.slow
def test_cfg2_full_size_properties():
    """cfg2 at its BASELINE size (1e6 x 64, 500 blocks): every sealed block
    orthonormal; L = 3.2e5 queries orthonormal, sign-canonical, and equal to the
    oracle's stitch of the GPU's own block factors."""
    cfg = workloads.CONFIGS["cfg2"]
    raw = workloads.generate("cfg2")
    g = z.BlockStore(cfg.b, cfg.c, policy=fixed(cfg.k))
    g.append(raw)
    assert g.sealed_count() == 500 and g.total_rows() == cfg.t
    blocks = {}
    for i in range(0, 500, 7):
        f = g.block(i)
        assert f.rank() == cfg.k and defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
    snap = g.snapshot()
    L = 320_000
    for t0 in workloads.query_offsets(cfg.t, L, 3, seed=42):
        t0 = int(t0)
        ans = z.range_query(snap, t0, t0 + L - 1, fixed(cfg.k)).factors
        assert ans.left_rows() == L and ans.rank() == cfg.k
        assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8
        for j in range(cfg.k):
            assert ans.v[int(np.argmax(np.abs(ans.v[:, j]))), j] >= 0
        S, E = t0 // cfg.b, (t0 + L - 1) // cfg.b
        for i in range(S, E + 1):
            if i not in blocks:
                blocks[i] = as_oracle(g.block(i))
        ref = oracle_query_from_blocks(blocks, cfg.b, t0, t0 + L - 1, cfg.k)
        assert_parity(ans, ref, what=f"cfg2 full L=3.2e5 at {t0}")


def test_host_pipelined_append_is_atomic_and_exact():
    """Large host appends are cut into chunks whose copies overlap the
    factorisation of earlier chunks. The result equals a device-input append
    bit for bit, and a rejected batch (non-finite row in the LAST chunk, after
    earlier chunks were already factorised) leaves the store and its snapshots
    unchanged (store.hpp:41-50 check_row; batch atomicity)."""
    b, c, k = 64, 16, 6
    rng = np.random.default_rng(77)
    raw = rng.standard_normal((300 * b + 37, c)) @ np.diag(np.linspace(5, 0.3, c))
    head = np.ascontiguousarray(raw[:123])
    body = np.ascontiguousarray(raw[123:])
    st = z.BlockStore(b, c, policy=fixed(k))
    st.append(head)
    snap = st.snapshot()
    q_before = z.range_query(snap, 10, 100, fixed(k)).factors
    bad = body.copy()
    bad[-50, 3] = np.inf
    with pytest.raises(z.InvalidInputError):
        st.append(bad)
    assert st.total_rows() == 123 and st.sealed_count() == 1
    q_again = z.range_query(snap, 10, 100, fixed(k)).factors
    assert np.array_equal(q_before.u, q_again.u) and np.array_equal(q_before.v, q_again.v)
    st.append(body)
    assert st.total_rows() == raw.shape[0] and st.sealed_count() == 300
    ref = z.BlockStore(b, c, policy=fixed(k))
    L = _capi.lib()
    ptr = C.c_void_p()
    full = np.ascontiguousarray(raw)
    assert L.zsvd_device_alloc(full.nbytes, 0, C.byref(ptr)) == 0
    try:
        assert L.zsvd_memcpy(ptr, full.ctypes.data, full.nbytes, None) == 0
        assert L.zsvd_stream_sync(None) == 0
        ref.append_ptr(ptr.value, full.shape[0], c, _capi.MEM_DEVICE)
    finally:
        L.zsvd_device_free(ptr)
    for i in list(range(0, 300, 13)) + [299]:
        a, e = st.block(i), ref.block(i)
        assert np.array_equal(a.u, e.u) and np.array_equal(a.sigma, e.sigma) and np.array_equal(a.v, e.v), i
    r = O.Store(b, c, 1.0, policy=O.FIXED_RANK, k=k, mode=O.INCREMENTAL)
    r.append(raw)
    for a0, a1 in [(0, raw.shape[0] - 1), (100, 5000), (19000, 19236)]:
        assert_parity(z.range_query(st, a0, a1, fixed(k)).factors, r.range_query(a0, a1), what=f"[{a0},{a1}]")
