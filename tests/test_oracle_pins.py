"""Pins the CPU oracle (oracle/) to the reference's own tests.

The reference cannot be built here (Eigen3 / GoogleTest absent), so the oracle
is pinned by re-running the reference suites' assertions — known answers and
properties, at the reference's own tolerances — on bit-identical inputs
(tests/golden, replayed std::mt19937 streams).  Incremental mode is the
reference's row-by-row algorithm (store.hpp); direct mode is the GPU design.
"""
import math

import numpy as np
import pytest

import golden
import oracle as O
from parity import defect, reconstruction_error, rel_fro_error, reconstruct

MODES = [O.INCREMENTAL, O.DIRECT]


def store_from(raw, b, xi, mode=O.INCREMENTAL, policy=O.ENERGY, k=0):
    s = O.Store(b, raw.shape[1], xi, policy=policy, k=k, mode=mode)
    s.append(raw)
    return s


# ------------------------------------------------------------- svd_test.cpp
def test_thin_svd_known_answers():  # svd_test.cpp:26-47, 136-150
    f = O.thin_svd(np.eye(2))
    assert f.rank == 2 and abs(f.s[0] - 1) < 1e-12 and abs(f.s[1] - 1) < 1e-12
    assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
    f = O.thin_svd(np.array([[3.0, 0], [0, 2]]))
    assert abs(f.s[0] - 3) < 1e-12 and abs(f.s[1] - 2) < 1e-12
    f = O.thin_svd(np.array([[1.0, 2], [2, 4]]))
    assert f.rank == 1 and abs(f.s[0] - 5) < 1e-12
    r2 = 1 / math.sqrt(2)
    f = O.thin_svd(np.array([[3 * r2, r2], [3 * r2, -r2]]))
    assert f.rank == 2 and abs(f.s[0] - 3) < 1e-12 and abs(f.s[1] - 1) < 1e-12
    t = O.truncate(f, O.ENERGY, 0.9)
    assert t.rank == 1 and abs(t.s[0] - 3) < 1e-12
    z = O.thin_svd(np.zeros((4, 3)))
    assert z.rank == 0 and z.u.shape == (4, 0) and z.v.shape == (3, 0)


def test_thin_svd_rejects():  # svd_test.cpp:48-58
    a = np.zeros((2, 2))
    a[0, 0] = np.nan
    with pytest.raises(O.OracleError):
        O.thin_svd(a)
    with pytest.raises(O.OracleError):
        O.thin_svd(np.zeros((0, 3)))


def test_random_shapes():  # svd_test.cpp:67-85
    for c in golden.cases("svd_random_shapes"):
        a = c["a"]
        f = O.thin_svd(a)
        assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
        assert np.all(np.diff(f.s) <= 0) and (f.rank == 0 or f.s[-1] >= 0)
        assert rel_fro_error(a, reconstruct(f)) <= 1e-8


def test_permutation_and_padding_invariance():  # svd_test.cpp:87-134
    for c in golden.cases("svd_row_permutation"):
        sa, sb = O.thin_svd(c["a"]).s, O.thin_svd(c["shuffled"]).s
        assert sa.shape == sb.shape
        assert np.all(np.abs(sa - sb) <= 1e-10 * max(1.0, sa[0]))
    for c in golden.cases("svd_zero_padding"):
        sa, sb = O.thin_svd(c["a"]).s, O.thin_svd(c["padded"]).s
        assert sa.shape == sb.shape
        assert np.all(np.abs(sa - sb) <= 1e-10 * max(1.0, sa[0]))


def test_truncate_minimality_and_budget():  # svd_test.cpp:177-222
    for c in golden.cases("truncate_minimality"):
        f = O.thin_svd(c["a"])
        xi = c["xi"]
        t = O.truncate(f, O.ENERGY, xi)
        assert t.rank >= 1
        total = np.sum(f.s ** 2)
        cum = np.sum(f.s[:t.rank] ** 2)
        assert cum / total >= xi
        if t.rank > 1:
            assert (cum - f.s[t.rank - 1] ** 2) / total < xi
    for c in golden.cases("truncate_energy_bound"):
        t = O.truncate(O.thin_svd(c["a"]), O.ENERGY, c["xi"])
        assert reconstruction_error(c["a"], t) <= 1 - c["xi"] + 1e-12


def test_truncate_edges():  # svd_test.cpp:152-176
    f = O.thin_svd(golden.case("svd_misc", "threshold_one")["a"])
    assert O.truncate(f, O.ENERGY, 1.0).rank == f.rank
    zero = O.Factors(np.array([[1.0], [0], [0]]), np.array([0.0]), np.array([[1.0], [0]]))
    t = O.truncate(zero, O.ENERGY, 0.98)
    assert t.rank == 0 and t.u.shape == (3, 0) and t.v.shape == (2, 0)
    for bad in (0.0, -0.5, 1.5):
        with pytest.raises(O.OracleError):
            O.truncate(zero, O.ENERGY, bad)
    # FIXED_RANK keeps min(k, r)
    f = O.thin_svd(np.diag([5.0, 4, 3, 2]))
    assert O.truncate(f, O.FIXED_RANK, 1.0, 2).rank == 2
    assert O.truncate(f, O.FIXED_RANK, 1.0, 9).rank == 4


def test_defect_and_sign():  # svd_test.cpp:245-285
    assert O.orthonormality_defect(np.eye(2)) == 0.0
    assert abs(O.orthonormality_defect(np.diag([1.0, 2.0])) - 3.0) <= 1e-15
    with pytest.raises(O.OracleError):
        O.orthonormality_defect(np.zeros((2, 3)))
    f = O.Factors(np.array([[1.0], [0]]), np.array([2.0]), np.array([[-1.0], [0]]))
    c = O.canonical_sign(f)
    assert c.v[0, 0] == 1.0 and c.u[0, 0] == -1.0
    for case in golden.cases("svd_misc"):
        if case["name"] != "canonical":
            continue
        f = O.thin_svd(case["a"])
        once = O.canonical_sign(f)
        twice = O.canonical_sign(once)
        assert np.array_equal(once.u, twice.u) and np.array_equal(once.v, twice.v)
        assert np.array_equal(reconstruct(once), reconstruct(f))


# ----------------------------------------------------------- store_test.cpp
def test_repeated_row_sigma():  # store_test.cpp:85-94
    b = O.open_block_from_row([1.0, 2, 2])
    b = O.incremental_update(b, 1, [1.0, 2, 2], 4)
    assert b.rank == 1 and abs(b.s[0] - 4.242640687119285) <= 1e-12


def test_zero_row_and_first_row():  # store_test.cpp:47-55, 96-110
    b = O.open_block_from_row([1.0, 2, 2])
    sig = b.s.copy()
    b2 = O.incremental_update(b, 1, [0.0, 0, 0], 4)
    assert np.allclose(b2.s, sig, atol=1e-12, rtol=0)
    assert np.all(np.abs(b2.u[1]) <= 1e-12)
    for mode in MODES:
        s = O.Store(4, 3, 0.98, mode=mode)
        s.append([0.0, 0, 0])
        assert s.open_rows == 1 and s.block(0).rank == 0 and s.total_rows == 1


def test_incremental_matches_direct_and_full_contract():  # store_test.cpp:112-127
    raw = golden.case("store_cases", "incremental_vs_direct")["raw"]
    b = O.open_block_from_row(raw[0])
    b = O.incremental_update(b, 1, raw[1], 3)
    b = O.incremental_update(b, 2, raw[2], 3)
    assert rel_fro_error(reconstruct(O.thin_svd(raw)), reconstruct(b)) <= 1e-8
    one = O.open_block_from_row([1.0, 0])
    with pytest.raises(O.OracleError) as e:
        O.incremental_update(one, 1, [1.0, 0], 1)
    assert e.value.code == O.LOGIC_ERROR


def test_reorthonormalize_clean_and_repair():  # store_test.cpp:129-168
    clean = O.open_block_from_row([1.0, 2, 2])
    same = O.reorthonormalize(clean)
    assert np.array_equal(same.u, clean.u) and np.array_equal(same.s, clean.s)
    rng = np.random.default_rng(53)
    raw = rng.uniform(-1, 1, (6, 4))
    b = O.open_block_from_row(raw[0])
    for i in range(1, 6):
        b = O.incremental_update(b, i, raw[i], 8)
    b.u += rng.uniform(-1e-7, 1e-7, b.u.shape)
    assert 1e-10 < defect(b.u) < 1e-5
    before = reconstruct(b)
    fixed = O.reorthonormalize(b)
    assert defect(fixed.u) <= 1e-10
    assert rel_fro_error(before, reconstruct(fixed)) <= 1e-9


@pytest.mark.parametrize("mode", MODES)
def test_store_cases(mode):  # store_test.cpp:37-83, 201-259
    c = golden.case("store_cases", "full_block_seals")
    s = store_from(c["raw"], 6, 0.98, mode)
    assert s.sealed_count == 1 and s.open_rows == 0 and s.total_rows == 6
    c = golden.case("store_cases", "rank_one_stream")
    s = store_from(c["raw"], 8, 0.98, mode)
    assert s.sealed_count == 2 and s.block(0).rank == 1 and s.block(1).rank == 1
    c = golden.case("store_cases", "sealed_orthonormal")
    s = store_from(c["raw"], 10, 0.95, mode)
    assert s.sealed_count == 4
    for i in range(4):
        f = s.block(i)
        assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
    c = golden.case("store_cases", "partial_tail")
    s = store_from(c["raw"], 4, 0.98, mode)
    assert s.sealed_count == 2 and s.open_rows == 2 and s.total_rows == 10
    assert rel_fro_error(c["raw"][8:10], reconstruct(s.block(2))) <= 1e-9
    s = O.Store(4, 3, 0.98, mode=mode)
    with pytest.raises(O.OracleError):
        s.append([1.0, 2])
    with pytest.raises(O.OracleError):
        s.append([1.0, 2, np.nan])
    assert s.total_rows == 0


def test_open_block_defect_bounded():  # store_test.cpp:214-223
    raw = golden.case("store_cases", "open_defect_bounded")["raw"]
    s = O.Store(300, 4, 1.0, mode=O.INCREMENTAL)
    for i in range(299):
        s.append(raw[i])
        assert defect(s.block(0).u) <= 1e-8


@pytest.mark.parametrize("mode", MODES)
def test_sealed_energy_budget(mode):  # store_test.cpp:173-199
    for c in golden.cases("store_energy_budget"):
        raw, xi, b = c["raw"], c["xi"], c["b"]
        s = store_from(raw, b, xi, mode)
        assert s.sealed_count == 1
        rec = reconstruct(s.block(0))
        num, den = np.sum((raw - rec) ** 2), np.sum(raw ** 2)
        if xi == 1.0:
            assert math.sqrt(num / den) <= 1e-8
        else:
            assert num / den <= 1 - xi + 1e-9


# ----------------------------------------------------------- query_test.cpp
def test_trim_cases():  # query_test.cpp:47-90
    blk = O.thin_svd(golden.case("trim_stitch_cases", "trim_no_elimination")["a"])
    t = O.trim_block(blk, 0, 7, O.ENERGY, 1.0)
    assert rel_fro_error(reconstruct(blk), reconstruct(t)) <= 1e-10 and t.u.shape[0] == 8
    blk = O.thin_svd(golden.case("trim_stitch_cases", "trim_single_row")["a"])
    rec = reconstruct(blk)
    for j in (0, 3, 7):
        t = O.trim_block(blk, j, j, O.ENERGY, 1.0)
        assert t.rank == 1 and abs(t.s[0] - np.linalg.norm(rec[j])) <= 1e-10
    raw = golden.case("trim_stitch_cases", "trim_rank_two_half")["a"]
    blk = O.thin_svd(raw)
    assert blk.rank == 2
    t = O.trim_block(blk, 6, 11, O.ENERGY, 1.0)
    assert rel_fro_error(reconstruct(blk)[6:12], reconstruct(t)) <= 1e-9
    blk = O.thin_svd(golden.case("trim_stitch_cases", "trim_bad_ranges")["a"])
    for args in ((3, 2, 1.0), (0, 6, 1.0), (0, 5, 0.0)):
        with pytest.raises(O.OracleError) as e:
            O.trim_block(blk, args[0], args[1], O.ENERGY, args[2])
        assert e.value.code == O.INVALID_PARAMETER
    empty = O.Factors(np.zeros((6, 0)), np.zeros(0), np.zeros((3, 0)))
    t = O.trim_block(empty, 1, 4, O.ENERGY, 1.0)
    assert t.rank == 0 and t.u.shape == (4, 0) and t.v.shape == (3, 0)


def test_stitch_cases():  # query_test.cpp:92-136
    part = O.thin_svd(golden.case("trim_stitch_cases", "stitch_single_part")["a"])
    assert rel_fro_error(reconstruct(part), reconstruct(O.stitch([part]))) <= 1e-10
    c = golden.case("trim_stitch_cases", "stitch_two_parts")
    st = O.stitch([O.thin_svd(c["a"]), O.thin_svd(c["b"])])
    raw = np.vstack([c["a"], c["b"]])
    assert rel_fro_error(raw, reconstruct(st)) <= 1e-8
    assert defect(st.u) <= 1e-10 and defect(st.v) <= 1e-10
    ref = O.thin_svd(raw)
    assert st.rank == ref.rank and np.all(np.abs(st.s - ref.s) <= 1e-8 * ref.s[0])
    b1 = golden.case("trim_stitch_cases", "stitch_zero_part")["a"]
    empty = O.Factors(np.zeros((4, 0)), np.zeros(0), np.zeros((3, 0)))
    rec = reconstruct(O.stitch([O.thin_svd(b1), empty]))
    assert rec.shape[0] == 9 and rel_fro_error(b1, rec[:5]) <= 1e-9 and np.all(np.abs(rec[5:]) <= 1e-12)
    e2 = O.stitch([O.Factors(np.zeros((3, 0)), np.zeros(0), np.zeros((2, 0))),
                   O.Factors(np.zeros((4, 0)), np.zeros(0), np.zeros((2, 0)))])
    assert e2.rank == 0 and e2.u.shape[0] == 7
    c = golden.case("trim_stitch_cases", "stitch_mismatch")
    with pytest.raises(O.OracleError) as e:
        O.stitch([O.thin_svd(c["a"]), O.thin_svd(c["b"])])
    assert e.value.code == O.INVALID_INPUT
    with pytest.raises(O.OracleError) as e:
        O.stitch([])
    assert e.value.code == O.INVALID_PARAMETER


@pytest.mark.parametrize("mode", MODES)
def test_range_cases(mode):  # query_test.cpp:146-287
    c = golden.case("range_cases", "full_range")
    s = store_from(c["raw"], 5, 1.0, mode)
    a = s.range_query(0, 19)
    assert a.u.shape[0] == 20 and rel_fro_error(c["raw"], reconstruct(a)) <= 1e-6
    c = golden.case("range_cases", "block_aligned")
    s = store_from(c["raw"], 4, 1.0, mode)
    direct = O.stitch([s.block(1), s.block(2)])
    assert rel_fro_error(reconstruct(direct), reconstruct(s.range_query(4, 11))) <= 1e-9
    c = golden.case("range_cases", "single_row")
    s = store_from(c["raw"], 4, 1.0, mode)
    for j in (0, 3, 5, 11):
        a = s.range_query(j, j)
        assert a.u.shape[0] == 1 and a.rank == 1 and abs(a.s[0] - np.linalg.norm(c["raw"][j])) <= 1e-8
    c = golden.case("range_cases", "bad_ranges")
    s = store_from(c["raw"], 4, 1.0, mode)
    for (a, b, xi, code) in ((3, 2, 1.0, O.RANGE_ERROR), (0, 8, 1.0, O.RANGE_ERROR),
                             (0, 3, 0.0, O.INVALID_PARAMETER)):
        with pytest.raises(O.OracleError) as e:
            s.range_query(a, b, xi)
        assert e.value.code == code
    empty = O.Store(4, 3, 1.0, mode=mode)
    with pytest.raises(O.OracleError):
        empty.range_query(0, 0)
    c = golden.case("range_cases", "resolve")
    s = store_from(c["raw"], 4, 1.0, mode)
    r = s.resolve(5, 13)
    assert (r["start_block"], r["end_block"], r["skip_front"], r["keep_front"], r["keep_back"],
            r["skip_back"]) == (1, 3, 1, 3, 2, 0)


@pytest.mark.parametrize("mode", MODES)
def test_exhaustive_open_tail(mode):  # query_test.cpp:195-216
    raw = golden.case("range_cases", "exhaustive_open_tail")["raw"]
    s = store_from(raw, 4, 1.0, mode)
    assert s.open_rows > 0
    for a in range(14):
        for b in range(a, 14):
            ans = s.range_query(a, b)
            sl = raw[a:b + 1]
            assert ans.u.shape[0] == b - a + 1
            assert rel_fro_error(sl, reconstruct(ans)) <= 1e-6
            ref = O.thin_svd(sl)
            assert ans.rank == ref.rank
            assert np.all(np.abs(ans.s - ref.s) <= 1e-6 * ref.s[0])


@pytest.mark.parametrize("mode", MODES)
def test_lossy_and_signed(mode):  # query_test.cpp:218-270
    for c in golden.cases("range_cases"):
        if c.get("name") == "lossy_budget":
            s = store_from(c["raw"], 20, c["xi"], mode)
            for a, b in c["ranges"]:
                ans = s.range_query(a, b, c["xi"])
                assert reconstruction_error(c["raw"][a:b + 1], ans) <= 2 * (1 - c["xi"]) + 1e-6
        if c.get("name") == "orthonormal_signed":
            s = store_from(c["raw"], 8, 0.98, mode)
            for a, b in c["ranges"]:
                ans = s.range_query(a, b, 0.98)
                assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8
                assert np.all(np.diff(ans.s) <= 0)
                for j in range(ans.rank):
                    piv = int(np.argmax(np.abs(ans.v[:, j])))
                    assert ans.v[piv, j] >= 0


# -------------------------------------------------------- acceptance_test.cpp
@pytest.mark.parametrize("mode", MODES)
def test_c1_exact_regime(mode):  # acceptance_test.cpp:106-136
    raw = golden.cases("acceptance_c1")[0]["raw"]
    s = store_from(raw, 8, 1.0, mode)
    assert s.sealed_count == 4
    checked = 0
    for a in range(32):
        for b in range(a, 32):
            ans = s.range_query(a, b)
            sl = raw[a:b + 1]
            assert rel_fro_error(sl, reconstruct(ans)) <= 1e-6
            ref = O.thin_svd(sl)
            assert ans.rank == ref.rank
            assert np.all(np.abs(ans.s - ref.s) <= 1e-6 * ref.s)
            checked += 1
    assert checked == 528


def test_c2_lossy_budget():  # acceptance_test.cpp:140-170
    for c in golden.cases("acceptance_c2"):
        xi = c["xi"]
        s = store_from(c["raw"], 100, xi, O.DIRECT)
        for a, b in c["ranges"][:60]:
            ans = s.range_query(a, b, xi)
            assert reconstruction_error(c["raw"][a:b + 1], ans) <= 2 * (1 - xi) + 1e-6


def test_c6_incremental_equals_batch():  # acceptance_test.cpp:304-320
    for c in golden.cases("acceptance_c6"):
        raw, b = c["raw"], c["b"]
        s = store_from(raw, b, 1.0, O.INCREMENTAL)
        assert s.sealed_count == 1
        assert rel_fro_error(reconstruct(O.thin_svd(raw)), reconstruct(s.block(0))) <= 1e-8


@pytest.mark.parametrize("mode", MODES)
def test_c9_orthonormality(mode):  # acceptance_test.cpp:463-503
    for c in golden.cases("acceptance_c9"):
        raw, b, xi = c["raw"], c["b"], c["xi"]
        s = store_from(raw, b, xi, mode)
        for i in range(s.sealed_count):
            f = s.block(i)
            assert defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
        t = O.trim_block(s.block(0), 1, b - 2, O.ENERGY, xi)
        assert defect(t.u) <= 1e-8 and defect(t.v) <= 1e-8
        st = O.stitch([s.block(0), s.block(1)], O.ENERGY, xi)
        assert defect(st.u) <= 1e-8 and defect(st.v) <= 1e-8
        for a, e in c["ranges"]:
            ans = s.range_query(a, e, xi)
            assert defect(ans.u) <= 1e-8 and defect(ans.v) <= 1e-8


def test_incremental_vs_direct_on_baseline_like_blocks():
    """the reference's row-by-row algorithm and the direct
    block SVD agree far inside the 1e-9 bar on cfg1-like data."""
    from paper_1805_00754_b200 import workloads
    from parity import assert_parity
    raw = workloads.generate("cfg1", rows=2000)
    inc = store_from(raw, 1000, 1.0, O.INCREMENTAL, O.FIXED_RANK, 10)
    dire = store_from(raw, 1000, 1.0, O.DIRECT, O.FIXED_RANK, 10)
    for i in range(2):
        full = O.thin_svd(raw[i * 1000:(i + 1) * 1000])
        assert_parity(inc.block(i), dire.block(i), sigma_next=full.s[10], what=f"block {i}")
