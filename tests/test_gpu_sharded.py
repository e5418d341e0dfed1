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


def test_nccl_sharded_query_single_rank_is_the_single_store_query():
    """zsvd_sharded_range_query over a one-rank NCCL communicator: the Gram
    exchange is the identity, so the answer equals the single-store Gram stitch
    bit for bit; energy truncation falls back (UnsupportedError) to the band
    path and still matches."""
    from paper_1805_00754_b200.sharded import NcclComm
    b, c, k = 64, 16, 6
    rng = np.random.default_rng(11)
    raw = rng.standard_normal((8 * b, c)) @ np.diag(np.linspace(4, 0.5, c))
    comm = NcclComm(0, 1, 0)
    st = ShardedStore(b, c, raw.shape[0], z.Truncation.fixed_rank(k), 0, 1, device=0, comm=comm)
    st.append_local(raw)
    single = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
    single.append(raw)
    for a, e in [(0, raw.shape[0] - 1), (10, 300), (5, 470)]:
        u, s, v, (lo, hi) = st._device_query(a, e)
        want = z.range_query(single, a, e).factors
        assert (lo, hi) == (a, e + 1)
        np.testing.assert_array_equal(s, want.sigma)
        np.testing.assert_array_equal(v, want.v)
        np.testing.assert_array_equal(u, want.u)
    # stacks shorter than c take the engine path on one device: the sharded call
    # says so (on every rank alike) and range_query gathers the parts instead
    for a, e in [(63, 64), (100, 130)]:
        with pytest.raises(z.UnsupportedError):
            st._device_query(a, e)
        u, s, v, (lo, hi) = st.range_query(a, e)
        assert_parity(z.SvdFactors(u, s, v), z.range_query(single, a, e).factors, what=f"fallback [{a},{e}]")
    est = ShardedStore(b, c, raw.shape[0], z.Truncation.energy(0.9), 0, 1, device=0, comm=comm)
    est.append_local(raw)
    with pytest.raises(z.UnsupportedError):
        est._device_query(0, 300)
    u, s, v, _ = est.range_query(0, 300)
    esingle = z.BlockStore(b, c, 0.9)
    esingle.append(raw)
    assert_parity(z.SvdFactors(u, s, v), z.range_query(esingle, 0, 300).factors, what="energy fallback")
    with pytest.raises(z.RangeError):
        st._device_query(0, raw.shape[0])


_TWO_RANK = r"""
import os, sys
import numpy as np
import torch.distributed as dist
sys.path[:0] = [os.environ["ZROOT"], os.path.join(os.environ["ZROOT"], "tests")]
import paper_1805_00754_b200 as z
from paper_1805_00754_b200.sharded import NcclComm, ShardedStore
from parity import assert_parity
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
b, c, k, rows = 64, 16, 6, 4 * 64
rng = np.random.default_rng(9)
raw = rng.standard_normal((world * rows, c)) @ np.diag(np.linspace(4, 0.5, c))
comm = NcclComm(rank, world, rank, dist)
st = ShardedStore(b, c, rows, z.Truncation.fixed_rank(k), rank, world, dist=dist, device=rank, comm=comm)
st.append_local(raw[rank * rows:(rank + 1) * rows])
for a, e in [(0, world * rows - 1), (10, 300), (250, 270), (63, 64), (100, 130)]:
    u, s, v, (lo, hi) = st.range_query(a, e)
    got = [None] * world
    dist.all_gather_object(got, (lo, u))
    if rank == 0:
        uu = np.vstack([x[1] for x in sorted(got, key=lambda x: x[0]) if x[1].shape[0]])
        single = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
        single.append(raw)
        assert_parity(z.SvdFactors(uu, s, v), z.range_query(single, a, e).factors, what=f"nccl [{a},{e}]")
dist.barrier()
print("ok", rank)
"""


def test_nccl_sharded_query_two_ranks(tmp_path):
    """Two processes on two GPUs, the Grams exchanged over NCCL (needs >= 2 GPUs)."""
    import os
    import subprocess
    import sys
    if z.device_count() < 2:
        pytest.skip("needs two GPUs (one process per GPU; NCCL rejects two ranks on one device)")
    script = tmp_path / "two_rank.py"
    script.write_text(_TWO_RANK)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ZROOT=root)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29533", str(script)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
