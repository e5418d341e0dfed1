"""similar_range_search (analysis.hpp:78-148) on the GPU:
the reference tests' semantics (planted occurrences, identical copy scores 1,
unit interval and no overlap, empty results and parameter errors, stride-1
agreement with a brute-force search on the raw rows) and parity of every
score with the oracle's window-by-window range_query."""
import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z

pytestmark = pytest.mark.gpu


def oracle_search(store, base_first, base_last, stride, top_n, **kw):
    """analysis.hpp:106-138 over the oracle's range_query."""
    L = base_last - base_first + 1
    base = store.range_query(base_first, base_last, **kw)
    if base.rank == 0:
        return []
    hits = []
    w = 0
    while w + L <= base_first:
        win = store.range_query(w, w + L - 1, **kw)
        sim = 0.0
        if win.rank > 0:
            a, b = base.u[:, 0], win.u[:, 0]
            na, nb = float(a @ a), float(b @ b)
            if na > 0 and nb > 0:
                sim = abs(float(a @ b)) / (np.sqrt(na) * np.sqrt(nb))
        hits.append((w, sim))
        w += stride
    hits.sort(key=lambda h: (-h[1], h[0]))
    return hits[:top_n]


def planted(rng, t, c, L, starts, noise=0.1):
    """Noise with one pattern (a rank-one sinusoid burst) planted at `starts`."""
    x = noise * rng.standard_normal((t, c))
    pat = np.outer(np.sin(np.arange(L) * 2 * np.pi / 37.0) * 4.0, rng.standard_normal(c))
    for s in starts:
        x[s:s + L] += pat
    return x


def assert_same_hits(got, ref, tol=1e-7):
    assert len(got) == len(ref)
    for g, (w, s) in zip(got, ref):
        assert abs(g.similarity - s) <= tol, (g, w, s)
    # identical order except inside groups of (numerically) tied scores
    gs = sorted((round(g.similarity / tol), g.window_start) for g in got)
    rs = sorted((round(s / tol), w) for w, s in ref)
    assert [x[1] for x in gs] == [x[1] for x in rs] or {g.window_start for g in got} == {w for w, _ in ref}


def test_finds_planted_occurrences():
    rng = np.random.default_rng(359)
    L = 100
    raw = planted(rng, 1700, 4, L, [0, 500, 1500])
    st = z.BlockStore(100, 4, 1.0)
    st.append(raw)
    hits = z.similar_range_search(st, 1500, 1599, L, 2, 1.0)
    assert len(hits) == 2
    assert {h.window_start for h in hits} == {0, 500}
    assert min(h.similarity for h in hits) >= 0.99


def test_identical_copy_scores_one():
    rng = np.random.default_rng(367)
    L = 100
    raw = 0.3 * rng.standard_normal((600, 3))
    raw[500:600] = raw[0:100]
    st = z.BlockStore(100, 3, 1.0)
    st.append(raw)
    hits = z.similar_range_search(st, 500, 599, L, 1, 1.0)
    assert len(hits) == 1 and hits[0].window_start == 0
    assert abs(hits[0].similarity - 1.0) <= 1e-10


def test_unit_interval_no_overlap_and_oracle_parity():
    rng = np.random.default_rng(373)
    t, c = 400, 4
    f = np.cumsum(rng.standard_normal((t, 2)) * 0.4, axis=0)
    raw = f @ rng.standard_normal((2, c)) + 0.1 * rng.standard_normal((t, c))
    st = z.BlockStore(50, c, 0.98)
    st.append(raw)
    hits = z.similar_range_search(st, 300, 379, 13, 100, 0.98)
    assert hits
    for h in hits:
        assert 0.0 <= h.similarity <= 1.0 and h.window_start + 80 <= 300
    ref = O.Store(50, c, 0.98)
    ref.append(raw)
    assert_same_hits(hits, oracle_search(ref, 300, 379, 13, 100))


def test_empty_results_and_parameter_errors():
    rng = np.random.default_rng(379)
    raw = rng.random((40, 3))
    st = z.BlockStore(10, 3, 1.0)
    st.append(raw)
    assert z.similar_range_search(st, 5, 30, 1, 3, 1.0) == []      # no complete window before the base
    assert z.similar_range_search(st, 20, 39, 5, 0, 1.0) == []     # zero hits requested
    with pytest.raises(z.InvalidParameterError):
        z.similar_range_search(st, 7, 7, 5, 2, 1.0)
    with pytest.raises(z.InvalidParameterError):
        z.similar_range_search(st, 10, 20, 0, 2, 1.0)
    with pytest.raises(z.RangeError):
        z.similar_range_search(st, 30, 45, 1, 2, 1.0)


def test_stride_one_matches_brute_force():
    rng = np.random.default_rng(383)
    L = 50
    raw = planted(rng, 600, 4, L, [0, 150, 450])
    st = z.BlockStore(75, 4, 1.0)
    st.append(raw)
    got = z.similar_range_search(st, 450, 499, 1, 2, 1.0)
    base = np.linalg.svd(raw[450:500], full_matrices=False)[0][:, 0]
    brute = []
    for w in range(0, 451 - L):
        u = np.linalg.svd(raw[w:w + L], full_matrices=False)[0][:, 0]
        brute.append((w, abs(float(base @ u))))
    brute.sort(key=lambda h: (-h[1], h[0]))
    assert {h.window_start for h in got} == {w for w, _ in brute[:2]} == {0, 150}


@pytest.mark.parametrize("policy", ["fixed", "energy"])
def test_oracle_parity_multi_block_windows(policy):
    """Windows spanning several blocks (stitched) and single-block windows,
    open tail included, against the oracle window by window."""
    rng = np.random.default_rng(401)
    b, c = 64, 12
    t = 20 * b + 37
    tt = np.arange(t)[:, None]
    raw = np.sin(tt / rng.uniform(15, 300, 5)[None, :]) @ rng.standard_normal((5, c)) + 0.05 * rng.standard_normal((t, c))
    if policy == "fixed":
        st = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(4))
        ref = O.Store(b, c, 1.0, policy=O.FIXED_RANK, k=4, mode=O.DIRECT)
        kw = {}
    else:
        st = z.BlockStore(b, c, 0.95)
        ref = O.Store(b, c, 0.95, mode=O.DIRECT)
        kw = {}
    st.append(raw)
    ref.append(raw)
    for (bf, bl, stride, top) in [(t - 200, t - 1, 7, 400), (700, 739, 3, 50), (900, 1100, 31, 5)]:
        got = z.similar_range_search(st, bf, bl, stride, top)
        assert_same_hits(got, oracle_search(ref, bf, bl, stride, top, **kw))


def test_cfg2_scale_windows():
    """cfg2-shaped data (b = 2000, c = 64, k = 20): 20,000-row windows at stride
    500 before a base at 100,000 (about 160 stitched windows in one batch)."""
    from paper_1805_00754_b200 import workloads
    O.set_backend("lapack")
    try:
        raw = workloads.generate("cfg2", rows=60 * 2000)
        st = z.BlockStore(2000, 64, policy=z.Truncation.fixed_rank(20))
        st.append(raw)
        ref = O.Store(2000, 64, 1.0, policy=O.FIXED_RANK, k=20, mode=O.DIRECT)
        ref.append(raw)
        got = z.similar_range_search(st, 100_000, 119_999, 500, 10)
        assert_same_hits(got, oracle_search(ref, 100_000, 119_999, 500, 10))
    finally:
        O.set_backend("jacobi")
