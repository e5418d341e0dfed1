"""Sharded store through the GPU backend: two ranks emulated as host threads on
one GPU (their kernels never wait on each other; the only exchange is a host
allgather), checked against the single-store GPU range_query and the oracle."""
import threading

import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z
from paper_1805_00754_b200.sharded import ShardedStore
from parity import assert_parity

pytestmark = pytest.mark.gpu


class ThreadDist:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world
        self.local = threading.local()

    def all_gather_object(self, out, obj):
        r = self.local.rank
        self.slots[r] = obj
        self.bar.wait()
        for i in range(self.world):
            out[i] = self.slots[i]
        self.bar.wait()


def test_sharded_gpu_matches_single_store():
    b, c, k, world, bpr = 64, 16, 6, 2, 4
    rng = np.random.default_rng(9)
    raw = rng.standard_normal((world * bpr * b, c)) @ np.diag(np.linspace(4, 0.5, c))
    rows = bpr * b
    d = ThreadDist(world)
    ranges = [(0, world * rows - 1), (10, 300), (100, 130), (250, 270), (255, 256), (63, 64), (400, 511)]
    results = [None] * world
    errors = []

    def run(rank):
        try:
            d.local.rank = rank
            st = ShardedStore(b, c, rows, z.Truncation.fixed_rank(k), rank, world, dist=d, device=0)
            st.append_local(raw[rank * rows:(rank + 1) * rows])
            results[rank] = [st.range_query(a, e) for a, e in ranges]
        except Exception as ex:  # pragma: no cover
            errors.append(ex)
            d.bar.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    single = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
    single.append(raw)
    ref = O.Store(b, c, 1.0, policy=O.FIXED_RANK, k=k, mode=O.INCREMENTAL)
    ref.append(raw)
    for qi, (a, e) in enumerate(ranges):
        pieces = sorted(((results[r][qi][3][0], results[r][qi][0]) for r in range(world)
                         if results[r][qi][3][1] > results[r][qi][3][0]), key=lambda x: x[0])
        u = np.vstack([p[1] for p in pieces])
        s, v = results[0][qi][1], results[0][qi][2]
        np.testing.assert_array_equal(s, results[1][qi][1])
        got = z.SvdFactors(u, s, v)
        assert u.shape[0] == e - a + 1
        assert_parity(got, z.range_query(single, a, e).factors, what=f"sharded vs single [{a},{e}]")
        assert_parity(got, ref.range_query(a, e), what=f"sharded vs oracle [{a},{e}]")
