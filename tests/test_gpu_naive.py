"""naive_range_svd and reconstruction_error on the GPU (analysis.hpp:20-66,
SURVEY 8(f) rank 3): the reference analysis_test cases and parity with the
oracle's reconstruct-then-SVD."""
import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z
from parity import assert_parity, rel_fro_error, reconstruct

pytestmark = pytest.mark.gpu


def empty(m, n):
    return z.SvdFactors(np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0)))


def test_reconstruction_error_cases():
    rng = np.random.default_rng(307)
    raw = rng.uniform(-1, 1, (8, 4))
    assert z.reconstruction_error(raw, z.thin_svd(raw)) <= 1e-12
    inv = 1.0 / np.sqrt(2.0)
    raw2 = np.array([[3 * inv, inv], [3 * inv, -inv]])
    f = z.truncate_rank(z.thin_svd(raw2), 0.9)
    assert f.rank() == 1
    assert abs(z.reconstruction_error(raw2, f) - 0.1) <= 1e-12
    raw3 = rng.uniform(-1, 1, (5, 3))
    assert z.reconstruction_error(raw3, empty(5, 3)) == 1.0
    f4 = z.thin_svd(rng.uniform(-1, 1, (4, 3)))
    assert np.isinf(z.reconstruction_error(np.zeros((4, 3)), f4))
    assert z.reconstruction_error(np.zeros((4, 3)), empty(4, 3)) == 0.0
    with pytest.raises(z.InvalidInputError):
        z.reconstruction_error(np.zeros((5, 3)), f4)
    with pytest.raises(z.InvalidInputError):
        z.reconstruction_error(np.zeros((4, 2)), f4)


def test_reconstruction_error_invariant_under_tied_sigma_remixing():
    f = z.SvdFactors(np.array([[1.0, 0], [0, 1], [0, 0]]), np.array([2.0, 2.0]), np.eye(2))
    raw = (f.u * f.sigma) @ f.v.T
    raw[0, 1] += 0.125
    raw[2, 0] -= 0.25
    base = z.reconstruction_error(raw, f)
    sw = z.SvdFactors(f.u[:, ::-1].copy(), f.sigma.copy(), f.v[:, ::-1].copy())
    assert abs(z.reconstruction_error(raw, sw) - base) <= 1e-12
    fl = z.SvdFactors(f.u * [-1, 1], f.sigma.copy(), f.v * [-1, 1])
    assert abs(z.reconstruction_error(raw, fl) - base) <= 1e-12


def oracle_naive(ref, b, first, last):
    """analysis.hpp:49-66 over the oracle's blocks."""
    rows = []
    S, E = first // b, last // b
    for i in range(S, E + 1):
        f = ref.block(i)
        blk = (f.u * f.s) @ f.v.T
        lo = first - S * b if i == S else 0
        hi = last - E * b if i == E else blk.shape[0] - 1
        rows.append(blk[lo:hi + 1])
    return O.thin_svd(np.vstack(rows))


def test_naive_agrees_with_oracle_on_exact_store():
    rng = np.random.default_rng(353)
    raw = rng.uniform(-1, 1, (18, 4))
    st = z.BlockStore(5, 4, 1.0)
    st.append(raw)
    snap = st.snapshot()
    for s, e in [(0, 17), (3, 12), (6, 6)]:
        naive = z.naive_range_svd(snap, s, e)
        exact = O.thin_svd(raw[s:e + 1])
        assert rel_fro_error(reconstruct(exact), reconstruct(naive)) <= 1e-8
    with pytest.raises(z.RangeError):
        z.naive_range_svd(snap, 5, 18)


@pytest.mark.parametrize("b,c,k", [(64, 12, 5), (100, 80, 8)])
def test_naive_parity_with_oracle(b, c, k):
    rng = np.random.default_rng(b + c)
    t = 6 * b + 21
    raw = rng.standard_normal((t, c)) @ np.diag(np.logspace(0, -1.5, c))
    st = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
    st.append(raw)
    ref = O.Store(b, c, 1.0, policy=O.FIXED_RANK, k=k, mode=O.DIRECT)
    ref.append(raw)
    for s, e in [(3, b + 7), (10, t - 1), (2 * b, 2 * b + 5)]:
        got = z.naive_range_svd(st, s, e)
        assert_parity(got, oracle_naive(ref, b, s, e), what=f"naive [{s},{e}]")
        err = z.reconstruction_error(raw[s:e + 1], got)
        ref_err = np.sum((raw[s:e + 1] - reconstruct(got)) ** 2) / np.sum(raw[s:e + 1] ** 2)
        assert abs(err - ref_err) <= 1e-12 * max(1.0, ref_err)
