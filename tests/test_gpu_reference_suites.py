"""The reference's own GoogleTest suites (svd_test, store_test, query_test,
acceptance C1/C2/C6/C9), restated against the GPU path through the C-ABI, on
the reference's own inputs (tests/golden), plus oracle parity on each case.

Reference tolerances are kept where the test asserts a property; the oracle
comparisons use the north_star bar (1e-9 sigma / reconstruction, 1e-7 rad)."""
import math

import numpy as np
import pytest

import golden
import oracle as O
import paper_1805_00754_b200 as z
from parity import (assert_parity, defect, rel_fro_error, reconstruct, reconstruction_error,
                    sigma_rel)

pytestmark = pytest.mark.gpu


def gstore(raw, b, xi=1.0, policy=None):
    s = z.BlockStore(b, raw.shape[1], xi, policy=policy)
    s.append(raw)
    return s


def ostore(raw, b, xi=1.0, mode=O.INCREMENTAL, policy=O.ENERGY, k=0):
    s = O.Store(b, raw.shape[1], xi, policy=policy, k=k, mode=mode)
    s.append(raw)
    return s


def osvd_next(a, k):
    s = O.thin_svd(a).s
    return s[k] if k < len(s) else 0.0


# ------------------------------------------------------------- svd_test.cpp
def test_thin_svd_known_answers():
    f = z.thin_svd(np.eye(2))
    assert f.rank() == 2 and abs(f.sigma[0] - 1) < 1e-12 and abs(f.sigma[1] - 1) < 1e-12
    assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
    f = z.thin_svd([[3.0, 0], [0, 2]])
    assert abs(f.sigma[0] - 3) < 1e-12 and abs(f.sigma[1] - 2) < 1e-12
    f = z.thin_svd([[1.0, 2], [2, 4]])
    assert f.rank() == 1 and abs(f.sigma[0] - 5) < 1e-12
    r2 = 1 / math.sqrt(2)
    f = z.thin_svd([[3 * r2, r2], [3 * r2, -r2]])
    assert f.rank() == 2 and abs(f.sigma[0] - 3) < 1e-12 and abs(f.sigma[1] - 1) < 1e-12
    t = z.truncate_rank(f, 0.9)
    assert t.rank() == 1 and abs(t.sigma[0] - 3) < 1e-12
    zf = z.thin_svd(np.zeros((4, 3)))
    assert zf.rank() == 0 and zf.left_rows() == 4 and zf.right_rows() == 3


def test_thin_svd_rejects():
    a = np.zeros((2, 2))
    a[0, 0] = np.nan
    with pytest.raises(z.InvalidInputError):
        z.thin_svd(a)
    with pytest.raises(z.InvalidInputError):
        z.thin_svd(np.zeros((0, 3)))
    with pytest.raises(z.InvalidInputError):
        z.thin_svd(np.zeros((3, 0)))


def test_random_shapes_and_oracle_parity():
    for c in golden.cases("svd_random_shapes"):
        a = c["a"]
        f = z.thin_svd(a)
        assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
        assert np.all(np.diff(f.sigma) <= 0)
        assert rel_fro_error(a, reconstruct(f)) <= 1e-8
        assert_parity(f, O.thin_svd(a), sigma_next=0.0, what=str(a.shape))


def test_invariances():
    for c in golden.cases("svd_row_permutation"):
        sa, sb = z.thin_svd(c["a"]).sigma, z.thin_svd(c["shuffled"]).sigma
        assert sa.shape == sb.shape and np.all(np.abs(sa - sb) <= 1e-10 * max(1.0, sa[0]))
    for c in golden.cases("svd_zero_padding"):
        sa, sb = z.thin_svd(c["a"]).sigma, z.thin_svd(c["padded"]).sigma
        assert sa.shape == sb.shape and np.all(np.abs(sa - sb) <= 1e-10 * max(1.0, sa[0]))


def test_truncate_properties():
    for c in golden.cases("truncate_minimality"):
        f = z.thin_svd(c["a"])
        t = z.truncate_rank(f, c["xi"])
        total = np.sum(f.sigma ** 2)
        cum = np.sum(f.sigma[:t.rank()] ** 2)
        assert t.rank() >= 1 and cum / total >= c["xi"]
        if t.rank() > 1:
            assert (cum - f.sigma[t.rank() - 1] ** 2) / total < c["xi"]
        assert t.rank() == O.truncate(O.thin_svd(c["a"]), O.ENERGY, c["xi"]).rank
    for c in golden.cases("truncate_energy_bound"):
        t = z.truncate_rank(z.thin_svd(c["a"]), c["xi"])
        assert reconstruction_error(c["a"], t) <= 1 - c["xi"] + 1e-12
    zero = z.SvdFactors(np.array([[1.0], [0], [0]]), np.array([0.0]), np.array([[1.0], [0]]))
    t = z.truncate_rank(zero, 0.98)
    assert t.rank() == 0 and t.left_rows() == 3 and t.right_rows() == 2
    for bad in (0.0, -0.5, 1.5):
        with pytest.raises(z.InvalidParameterError):
            z.truncate_rank(zero, bad)
    f = z.thin_svd(np.diag([5.0, 4, 3, 2]))
    assert z.truncate_rank(f, z.Truncation.fixed_rank(2)).rank() == 2


def test_canonical_sign():
    f = z.SvdFactors(np.array([[1.0], [0]]), np.array([2.0]), np.array([[-1.0], [0]]))
    c = z.canonical_sign(f)
    assert c.v[0, 0] == 1.0 and c.u[0, 0] == -1.0
    for case in golden.cases("svd_misc"):
        if case["name"] != "canonical":
            continue
        f = z.thin_svd(case["a"])
        once = z.canonical_sign(f)
        twice = z.canonical_sign(once)
        assert np.array_equal(once.u, twice.u) and np.array_equal(once.v, twice.v)
        assert np.array_equal(reconstruct(once), reconstruct(f))
        ref = O.canonical_sign(O.thin_svd(case["a"]))
        # same pivots -> same signs as the oracle's canonical form
        assert np.all(np.sign(np.sum(once.v * ref.v, axis=0)) > 0)


# ----------------------------------------------------------- store_test.cpp
def test_store_ctor_and_rejects():
    s = z.BlockStore(1000, 16, 0.98)
    assert s.total_rows() == 0 and s.sealed_count() == 0 and s.open() is None
    s = z.BlockStore(1, 1, 1.0)
    assert s.block_size() == 1 and s.num_columns() == 1
    for args in ((0, 5, 0.98), (5, 0, 0.98), (5, 5, 0.0), (5, 5, 1.5)):
        with pytest.raises(z.InvalidParameterError):
            z.BlockStore(*args)
    s = z.BlockStore(4, 3, 0.98)
    with pytest.raises(z.InvalidInputError):
        s.append([1.0, 2])
    with pytest.raises(z.InvalidInputError):
        s.append([1.0, 2, np.nan])
    with pytest.raises(z.InvalidInputError):  # whole batch rejected atomically
        s.append([[1.0, 2, 3], [np.inf, 0, 0]])
    assert s.total_rows() == 0


def test_store_known_answers():
    s = z.BlockStore(4, 3, 0.98)
    s.append([1.0, 2, 2])
    s.append([1.0, 2, 2])
    f = s.open()
    assert f.rank() == 1 and abs(f.sigma[0] - 4.242640687119285) <= 1e-12   # store_test.cpp:85-94
    s = z.BlockStore(4, 3, 0.98)
    s.append([0.0, 0, 0])
    assert s.open_rows() == 1 and s.open().rank() == 0 and s.total_rows() == 1  # :47-55
    s = z.BlockStore(4, 3, 0.98)
    s.append([1.0, 2, 2])
    sig = s.open().sigma.copy()
    s.append([0.0, 0, 0])
    f = s.open()
    assert np.allclose(f.sigma, sig, atol=1e-12, rtol=0) and np.all(np.abs(f.u[1]) <= 1e-12)  # :96-110


@pytest.mark.parametrize("label,b,xi", [("full_block_seals", 6, 0.98), ("rank_one_stream", 8, 0.98),
                                        ("sealed_orthonormal", 10, 0.95), ("partial_tail", 4, 0.98),
                                        ("incremental_vs_direct", 3, 1.0), ("from_parts", 4, 0.98)])
def test_store_cases_vs_oracle(label, b, xi):
    raw = golden.case("store_cases", label)["raw"]
    g = gstore(raw, b, xi)
    r = ostore(raw, b, xi)
    assert g.sealed_count() == r.sealed_count and g.total_rows() == r.total_rows
    assert g.open_rows() == r.open_rows
    for i in range(r.sealed_count + (1 if r.open_rows else 0)):
        fg, fr = g.block(i), r.block(i)
        assert defect(fg.u) <= 1e-10 and defect(fg.v) <= 1e-10
        lo = i * b
        nxt = osvd_next(raw[lo:lo + b], fr.rank)
        assert_parity(fg, fr, sigma_next=nxt, what=f"{label} block {i}")
    if label == "rank_one_stream":
        assert g.block(0).rank() == 1 and g.block(1).rank() == 1
    if label == "partial_tail":
        assert rel_fro_error(raw[8:10], reconstruct(g.open())) <= 1e-9


def test_open_block_defect_bounded():  # store_test.cpp:214-223
    raw = golden.case("store_cases", "open_defect_bounded")["raw"]
    s = z.BlockStore(300, 4, 1.0)
    for i in range(299):
        s.append(raw[i])
        if i % 23 == 0 or i == 298:
            assert defect(s.open().u) <= 1e-8


def test_sealed_energy_budget():  # store_test.cpp:173-199
    for c in golden.cases("store_energy_budget"):
        raw, xi, b = c["raw"], c["xi"], c["b"]
        s = gstore(raw, b, xi)
        assert s.sealed_count() == 1
        rec = reconstruct(s.block(0))
        num, den = np.sum((raw - rec) ** 2), np.sum(raw ** 2)
        if xi == 1.0:
            assert math.sqrt(num / den) <= 1e-8
        else:
            assert num / den <= 1 - xi + 1e-9
        assert s.block(0).rank() == ostore(raw, b, xi).block(0).rank


def test_snapshot_isolation():  # store_test.cpp:237-259
    raw = golden.case("store_cases", "snapshot")["raw"]
    s = z.BlockStore(4, 3, 1.0)
    s.append(raw[:6])
    snap = s.snapshot()
    assert snap.sealed_count == 1 and snap.total_rows == 6 and snap.open_rows == 2
    before = z.range_query(snap, 0, 5).factors
    s.append(raw[6:])
    assert s.sealed_count() == 3
    assert snap.sealed_count == 1 and snap.block_count() == 2 and snap.block_rows(1) == 2
    after = z.range_query(snap, 0, 5).factors
    assert np.array_equal(before.u, after.u) and np.array_equal(before.sigma, after.sigma)
    with pytest.raises(z.RangeError):
        z.range_query(snap, 0, 6)


# ----------------------------------------------------------- query_test.cpp
def test_trim_cases():
    blk = z.thin_svd(golden.case("trim_stitch_cases", "trim_no_elimination")["a"])
    t = z.trim_block(blk, 0, 7, 1.0)
    assert rel_fro_error(reconstruct(blk), reconstruct(t)) <= 1e-10 and t.left_rows() == 8
    blk = z.thin_svd(golden.case("trim_stitch_cases", "trim_single_row")["a"])
    rec = reconstruct(blk)
    for j in (0, 3, 7):
        t = z.trim_block(blk, j, j, 1.0)
        assert t.rank() == 1 and abs(t.sigma[0] - np.linalg.norm(rec[j])) <= 1e-10
    raw = golden.case("trim_stitch_cases", "trim_rank_two_half")["a"]
    blk = z.thin_svd(raw)
    assert blk.rank() == 2
    t = z.trim_block(blk, 6, 11, 1.0)
    assert rel_fro_error(reconstruct(blk)[6:12], reconstruct(t)) <= 1e-9
    blk = z.thin_svd(golden.case("trim_stitch_cases", "trim_bad_ranges")["a"])
    for a, b, xi in ((3, 2, 1.0), (0, 6, 1.0), (0, 5, 0.0)):
        with pytest.raises(z.InvalidParameterError):
            z.trim_block(blk, a, b, xi)
    empty = z.SvdFactors(np.zeros((6, 0)), np.zeros(0), np.zeros((3, 0)))
    t = z.trim_block(empty, 1, 4, 1.0)
    assert t.rank() == 0 and t.left_rows() == 4 and t.right_rows() == 3


def test_trim_parity_vs_oracle():
    rng = np.random.default_rng(5)
    for m, n in ((40, 6), (300, 20), (2000, 20), (9, 16), (1, 12)):
        a = rng.standard_normal((m, n)) @ np.diag(np.linspace(3, 0.5, n))
        fo = O.thin_svd(a)
        fg = z.thin_svd(a)
        assert_parity(fg, fo, sigma_next=0.0, what=f"thin_svd {m}x{n}")
        for lo, hi in ((0, m - 1), (m // 3, m - 1), (0, max(0, m // 2)), (m - 1, m - 1)):
            for xi in (1.0, 0.9):
                tg = z.trim_block(fg, lo, hi, xi)
                to = O.trim_block(fo, lo, hi, O.ENERGY, xi)
                assert tg.rank() == to.rank
                assert sigma_rel(tg.sigma, to.s) <= 1e-9
                assert rel_fro_error(reconstruct(to), reconstruct(tg)) <= 1e-9


def test_stitch_cases():
    part = z.thin_svd(golden.case("trim_stitch_cases", "stitch_single_part")["a"])
    assert rel_fro_error(reconstruct(part), reconstruct(z.stitch([part], 1.0))) <= 1e-10
    c = golden.case("trim_stitch_cases", "stitch_two_parts")
    st = z.stitch([z.thin_svd(c["a"]), z.thin_svd(c["b"])], 1.0)
    raw = np.vstack([c["a"], c["b"]])
    assert rel_fro_error(raw, reconstruct(st)) <= 1e-8
    assert defect(st.u) <= 1e-10 and defect(st.v) <= 1e-10
    ref = O.thin_svd(raw)
    assert st.rank() == ref.rank and np.all(np.abs(st.sigma - ref.s) <= 1e-8 * ref.s[0])
    b1 = golden.case("trim_stitch_cases", "stitch_zero_part")["a"]
    empty = z.SvdFactors(np.zeros((4, 0)), np.zeros(0), np.zeros((3, 0)))
    rec = reconstruct(z.stitch([z.thin_svd(b1), empty], 1.0))
    assert rec.shape[0] == 9 and rel_fro_error(b1, rec[:5]) <= 1e-9 and np.all(np.abs(rec[5:]) <= 1e-12)
    e2 = z.stitch([z.SvdFactors(np.zeros((3, 0)), np.zeros(0), np.zeros((2, 0))),
                   z.SvdFactors(np.zeros((4, 0)), np.zeros(0), np.zeros((2, 0)))], 1.0)
    assert e2.rank() == 0 and e2.left_rows() == 7
    c = golden.case("trim_stitch_cases", "stitch_mismatch")
    with pytest.raises(z.InvalidInputError):
        z.stitch([z.thin_svd(c["a"]), z.thin_svd(c["b"])], 1.0)
    with pytest.raises(z.InvalidParameterError):
        z.stitch([], 1.0)


def test_range_cases():
    c = golden.case("range_cases", "full_range")
    s = gstore(c["raw"], 5)
    a = z.range_query(s, 0, 19, 1.0)
    assert a.rows() == 20 and rel_fro_error(c["raw"], reconstruct(a.factors)) <= 1e-6
    c = golden.case("range_cases", "block_aligned")
    s = gstore(c["raw"], 4)
    direct = z.stitch([s.block(1), s.block(2)], 1.0)
    assert rel_fro_error(reconstruct(direct), reconstruct(z.range_query(s, 4, 11, 1.0).factors)) <= 1e-9
    c = golden.case("range_cases", "single_row")
    s = gstore(c["raw"], 4)
    for j in (0, 3, 5, 11):
        a = z.range_query(s, j, j, 1.0)
        assert a.rows() == 1 and a.rank() == 1
        assert abs(a.factors.sigma[0] - np.linalg.norm(c["raw"][j])) <= 1e-8
    c = golden.case("range_cases", "bad_ranges")
    s = gstore(c["raw"], 4)
    with pytest.raises(z.RangeError):
        z.range_query(s, 3, 2, 1.0)
    with pytest.raises(z.RangeError):
        z.range_query(s, 0, 8, 1.0)
    with pytest.raises(z.InvalidParameterError):
        z.range_query(s, 0, 3, 0.0)
    with pytest.raises(z.RangeError):
        z.range_query(z.BlockStore(4, 3, 1.0), 0, 0, 1.0)
    c = golden.case("range_cases", "resolve")
    s = gstore(c["raw"], 4)
    r = s.snapshot().resolve(5, 13)
    assert (r.start_block, r.end_block, r.skip_front, r.keep_front, r.keep_back, r.skip_back,
            r.length()) == (1, 3, 1, 3, 2, 0, 9)


def test_exhaustive_open_tail_vs_oracle():  # query_test.cpp:195-216
    raw = golden.case("range_cases", "exhaustive_open_tail")["raw"]
    g = gstore(raw, 4)
    r = ostore(raw, 4)
    snap = g.snapshot()
    for a in range(14):
        for b in range(a, 14):
            ans = z.range_query(snap, a, b, 1.0).factors
            sl = raw[a:b + 1]
            assert ans.left_rows() == b - a + 1
            assert rel_fro_error(sl, reconstruct(ans)) <= 1e-6
            ref = O.thin_svd(sl)
            assert ans.rank() == ref.rank and np.all(np.abs(ans.sigma - ref.s) <= 1e-6 * ref.s[0])
            assert_parity(ans, r.range_query(a, b), sigma_next=0.0, what=f"[{a},{b}]")


def test_lossy_budget_and_signed_outputs():
    for c in golden.cases("range_cases"):
        if c.get("name") == "lossy_budget":
            s = gstore(c["raw"], 20, c["xi"])
            snap = s.snapshot()
            for a, b in c["ranges"]:
                ans = z.range_query(snap, a, b, c["xi"]).factors
                assert reconstruction_error(c["raw"][a:b + 1], ans) <= 2 * (1 - c["xi"]) + 1e-6
        if c.get("name") == "orthonormal_signed":
            s = gstore(c["raw"], 8, 0.98)
            snap = s.snapshot()
            for a, b in c["ranges"]:
                ans = z.range_query(snap, a, b, 0.98).factors
                assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8
                assert np.all(np.diff(ans.sigma) <= 0)
                for j in range(ans.rank()):
                    piv = int(np.argmax(np.abs(ans.v[:, j])))
                    assert ans.v[piv, j] >= 0


# -------------------------------------------------------- acceptance_test.cpp
def test_c1_exact_regime_all_528_ranges():
    raw = golden.cases("acceptance_c1")[0]["raw"]
    g = gstore(raw, 8)
    r = ostore(raw, 8)
    assert g.sealed_count() == 4
    snap = g.snapshot()
    n = 0
    for a in range(32):
        for b in range(a, 32):
            ans = z.range_query(snap, a, b, 1.0).factors
            sl = raw[a:b + 1]
            assert rel_fro_error(sl, reconstruct(ans)) <= 1e-6
            ref = O.thin_svd(sl)
            assert ans.rank() == ref.rank and np.all(np.abs(ans.sigma - ref.s) <= 1e-6 * ref.s)
            assert_parity(ans, r.range_query(a, b), sigma_next=0.0, what=f"C1 [{a},{b}]")
            n += 1
    assert n == 528


def test_c2_lossy_budget():
    for c in golden.cases("acceptance_c2"):
        xi = c["xi"]
        s = gstore(c["raw"], 100, xi)
        snap = s.snapshot()
        for a, b in c["ranges"]:
            ans = z.range_query(snap, a, b, xi).factors
            assert reconstruction_error(c["raw"][a:b + 1], ans) <= 2 * (1 - xi) + 1e-6


def test_c6_incremental_equals_batch():
    for c in golden.cases("acceptance_c6"):
        raw, b = c["raw"], c["b"]
        g = gstore(raw, b)
        assert g.sealed_count() == 1
        assert rel_fro_error(reconstruct(O.thin_svd(raw)), reconstruct(g.block(0))) <= 1e-8
        inc = ostore(raw, b).block(0)
        assert_parity(g.block(0), inc, sigma_next=0.0, what=f"C6 {raw.shape}")


def test_c9_orthonormality():
    for c in golden.cases("acceptance_c9"):
        raw, b, xi = c["raw"], c["b"], c["xi"]
        s = gstore(raw, b, xi)
        for i in range(s.sealed_count()):
            f = s.block(i)
            assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
        t = z.trim_block(s.block(0), 1, b - 2, xi)
        assert defect(t.u) <= 1e-8 and defect(t.v) <= 1e-8
        st = z.stitch([s.block(0), s.block(1)], xi)
        assert defect(st.u) <= 1e-8 and defect(st.v) <= 1e-8
        snap = s.snapshot()
        for a, e in c["ranges"]:
            ans = z.range_query(snap, a, e, xi).factors
            assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8
