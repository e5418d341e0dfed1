"""Wide path (64 < min(m, n) <= 1024, wide_engine.cu) against the oracle:
thin_svd shapes, rank-deficient input, c > 64 stores (blocks, open tail,
queries whose stitch is tall and whose stitch is wide), the energy policy,
and batch atomicity of host appends to a wide store.

The oracle runs in DIRECT mode (LAPACK dgesdd per block) for these widths:
its incremental mode would take minutes per block at c = 256, and
SURVEY 8(c) / C6 / store_test :112-121 justify direct == incremental."""
import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z
from paper_1805_00754_b200 import workloads
from parity import assert_parity, defect

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def lapack_oracle():
    O.set_backend("lapack")
    yield
    O.set_backend("jacobi")


def graded(rng, m, n, decades=2.0):
    return rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -decades, n))


@pytest.mark.parametrize("shape", [(600, 100), (100, 600), (700, 300), (300, 1024), (1100, 1024)])
def test_thin_svd_wide_shapes(shape):
    rng = np.random.default_rng(sum(shape))
    a = graded(rng, *shape)
    g = z.thin_svd(a)
    r = O.thin_svd(a)
    assert_parity(g, r, what=f"thin_svd {shape}")
    assert defect(g.u) <= 1e-10 and defect(g.v) <= 1e-10


def test_thin_svd_wide_rank_deficient():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((400, 30)) @ rng.standard_normal((30, 200))
    g = z.thin_svd(a)
    r = O.thin_svd(a)
    assert g.rank() == r.rank == 30
    assert_parity(g, r, what="rank-deficient 400x200")


def _store_pair(b, c, raw, policy, xi=1.0, k=0):
    if policy == O.FIXED_RANK:
        g = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
    else:
        g = z.BlockStore(b, c, xi)
    r = O.Store(b, c, xi, policy=policy, k=k, mode=O.DIRECT)
    g.append(raw)
    r.append(raw)
    return g, r


@pytest.mark.parametrize("b,c,k", [(300, 100, 12), (128, 256, 30)])
def test_wide_store_blocks_and_queries(b, c, k):
    rng = np.random.default_rng(b + c)
    t = 5 * b + 77
    base = np.sin(np.arange(t)[:, None] / rng.uniform(20, 400, 8)[None, :]) @ rng.standard_normal((8, c))
    raw = base + 0.05 * rng.standard_normal((t, c))
    g, r = _store_pair(b, c, raw, O.FIXED_RANK, k=k)
    assert g.sealed_count() == r.sealed_count == 5 and g.total_rows() == t
    for i in range(5):
        assert_parity(g.block(i), r.block(i), what=f"block {i}")
    snap = g.snapshot()
    # single block, two blocks, many blocks (stitch K = 3k..5k rows: wide when
    # K < c, tall otherwise), and ranges reaching into the open tail
    for a0, a1 in [(5, b - 3), (b - 10, b + 20), (17, 3 * b + 5), (0, t - 1), (2 * b + 1, t - 1)]:
        assert_parity(z.range_query(snap, a0, a1, z.Truncation.fixed_rank(k)).factors, r.range_query(a0, a1),
                      what=f"query [{a0}, {a1}]")


def test_wide_store_energy_policy():
    rng = np.random.default_rng(3)
    b, c = 200, 96
    raw = graded(rng, 3 * b + 50, c, decades=3.0)
    g, r = _store_pair(b, c, raw, O.ENERGY, xi=0.9)
    for i in range(3):
        assert_parity(g.block(i), r.block(i), what=f"energy block {i}")
    for a0, a1 in [(10, 150), (30, 2 * b + 40), (0, 3 * b + 49)]:
        assert_parity(z.range_query(g, a0, a1).factors, r.range_query(a0, a1), what=f"energy query [{a0}, {a1}]")


def test_cfg3_blocks_match_oracle():
    """Two cfg3 blocks (4000 x 256, k = 30) and queries across them."""
    cfg = workloads.CONFIGS["cfg3"]
    raw = workloads.generate("cfg3", rows=2 * cfg.b + 300)
    g, r = _store_pair(cfg.b, cfg.c, raw, O.FIXED_RANK, k=cfg.k)
    for i in range(2):
        f = g.block(i)
        assert f.rank() == cfg.k and defect(f.u) <= 1e-10 and defect(f.v) <= 1e-10
        assert_parity(f, r.block(i), what=f"cfg3 block {i}")
    for a0, a1 in [(100, 3900), (3000, 5000), (0, 2 * cfg.b + 299)]:
        assert_parity(z.range_query(g, a0, a1).factors, r.range_query(a0, a1), what=f"cfg3 [{a0}, {a1}]")


def test_wide_host_append_is_atomic():
    rng = np.random.default_rng(8)
    b, c = 150, 128
    raw = rng.standard_normal((4 * b, c))
    g = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(10))
    g.append(raw[:b + 10])
    bad = raw[b + 10:].copy()
    bad[-3, 7] = np.nan
    with pytest.raises(z.InvalidInputError):
        g.append(bad)
    assert g.total_rows() == b + 10 and g.sealed_count() == 1
    g.append(raw[b + 10:])
    r = O.Store(b, c, 1.0, policy=O.FIXED_RANK, k=10, mode=O.DIRECT)
    r.append(raw)
    for i in range(4):
        assert_parity(g.block(i), r.block(i), what=f"block {i}")
