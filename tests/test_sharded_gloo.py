"""Multi-rank logic of the sharded store (paper_1805_00754_b200/sharded.py) on
CPU: world_size 2 over gloo, each rank computing with the oracle backend; the
assembled answer must equal the single-store range_query (query.hpp:163-201)
on the same stream, row for row."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1805_00754_b200.sharded import Part, ShardedStore

B, C, K = 8, 5, 3
BLOCKS_PER_RANK = 3


class OracleBackend:
    """Oracle compute behind the same interface as sharded.GpuBackend."""

    def __init__(self, b, c, trunc):
        self.store = O.Store(b, c, 1.0, policy=O.FIXED_RANK, k=trunc, mode=O.INCREMENTAL)
        self.k = trunc

    def snapshot(self):
        return self.store.total_rows

    def block(self, i):
        return self.store.block(i)

    def trim(self, blk, lo, hi, trunc):
        return O.trim_block(blk, lo, hi, O.FIXED_RANK, 1.0, trunc)

    def to_part(self, f, with_u=True):
        return Part(f.u if with_u else None, f.s, f.v, f.u.shape[0])

    def stitch(self, parts, trunc):
        fs = [O.Factors(p.u if p.u is not None else np.zeros((0, p.s.shape[0])), p.s, p.v) for p in parts]
        return _Res(O.canonical_sign(O.stitch(fs, O.FIXED_RANK, 1.0, trunc)))

    def sign(self, f):
        return O.canonical_sign(f)


class _Res:
    def __init__(self, f):
        self.u, self.sigma, self.v = f.u, f.s, f.v


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, raw, ranges, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = BLOCKS_PER_RANK * B
    st = ShardedStore(B, C, rows, K, rank, world, backend_factory=lambda b, c, t: OracleBackend(b, c, t),
                      dist=dist)
    st.append_local(raw[rank * rows:(rank + 1) * rows])
    res = []
    for first, last in ranges:
        u, s, v, (lo, hi) = st.range_query(first, last)
        res.append((u, s, v, lo, hi))
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_query_equals_single_store():
    world = 2
    rng = np.random.default_rng(3)
    raw = rng.standard_normal((world * BLOCKS_PER_RANK * B, C))
    ranges = [(0, 47), (3, 44), (20, 30), (9, 14), (24, 31), (17, 40), (40, 40), (0, 7), (23, 24)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, raw, ranges, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.Store(B, C, 1.0, policy=O.FIXED_RANK, k=K, mode=O.INCREMENTAL)
    ref.append(raw)
    for qi, (first, last) in enumerate(ranges):
        want = ref.range_query(first, last)
        pieces = []
        for r in range(world):
            u, s, v, lo, hi = results[r][qi]
            np.testing.assert_array_equal(s, want.s)
            np.testing.assert_array_equal(v, want.v)
            if hi > lo:
                pieces.append((lo, u))
        pieces.sort(key=lambda x: x[0])
        u_all = np.vstack([p[1] for p in pieces])
        assert u_all.shape[0] == last - first + 1
        np.testing.assert_array_equal(u_all, want.u)


def _lag_worker(rank, world, port, raw, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = BLOCKS_PER_RANK * B
    st = ShardedStore(B, C, rows, K, rank, world, backend_factory=lambda b, c, t: OracleBackend(b, c, t),
                      dist=dist)
    # rank 0 lags: only its first 10 rows arrived; rank 1 is full
    n = 10 if rank == 0 else rows
    st.append_local(raw[rank * rows:rank * rows + n])
    res = []
    for first, last in [(5, 30), (9, 9), (12, 40), (0, 9)]:
        try:
            st.range_query(first, last)
            res.append("ok")
        except Exception as e:  # noqa: BLE001
            res.append(type(e).__name__)
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_lagging_rank_range_error_everywhere():
    """A range over rows a lagging lower rank has not received raises RangeError
    on every rank (no rank enters a collective the others skip)."""
    world = 2
    raw = np.random.default_rng(4).standard_normal((world * BLOCKS_PER_RANK * B, C))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lag_worker, args=(r, world, port, raw, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert results[r] == ["RangeError", "ok", "RangeError", "ok"], results[r]


def test_layout():
    st = ShardedStore.__new__(ShardedStore)
    st.rows_per_rank, st.rank = 24, 1
    assert st.owner_of_row(23) == 0 and st.owner_of_row(24) == 1
    assert st.local_range() == (24, 48)
    with pytest.raises(ValueError):
        ShardedStore(8, 5, 20, 3, 0, 1, backend_factory=lambda b, c, t: OracleBackend(b, c, t))
