"""Block-range sharding over ranks: one process per GPU.

Storage shards with no collective: rank r owns the global rows
[r * rows_per_rank, (r + 1) * rows_per_rank) (a multiple of the block size),
i.e. a contiguous range of whole blocks, and runs its own BlockStore on its own
device.

A range query [first, last] over the global stream runs, when every rank holds
a GPU store and the stitch is a Gram stitch (FIXED_RANK, c <= 64: the BASELINE
configs' narrow path), in libzsvd (zsvd_sharded_range_query): each rank forms
the Gram of its share of the stitched stack on its GPU, the c x c Grams are
all-gathered over NCCL (NcclComm, one communicator per rank) and added in rank
order, the stitch SVD runs replicated, and each rank writes the U rows of its
own share; no factor leaves the devices.

Otherwise (energy truncation, c > 64, a spread spectrum: UnsupportedError from
that call, or the CPU test backends) it follows range_query (query.hpp:163-201)
exactly, distributed:
  1. the owner of block S trims the head, the owner of block E trims the tail
     (query.hpp:175-178); interior blocks are used as stored;
  2. every rank allgathers the parts' (rank k_p, sigma_p, V_p) — the stacked
     diag(sigma) V^T bands are tiny (k x c per block) — in global part order;
  3. every rank runs the same stitch (query.hpp:95-144) on the full part list,
     with its own parts carrying their U rows and remote parts row-less, so it
     gets the replicated (sigma, V) and the U rows of its own range only;
  4. canonical_sign (query.hpp:190) is decided by V, identical everywhere.
A single-block range (S == E) is one trim on the owner, broadcast.

The collectives are torch.distributed (NCCL on GPUs, gloo in the CPU tests);
the per-rank compute goes through a backend — GpuBackend (libzsvd.so) in the
product; tests inject an oracle-backed one to check the distributed logic.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np


@dataclass
class Part:
    """One stitched part: U rows (possibly none on remote ranks), sigma, V."""
    u: Optional[np.ndarray]
    s: np.ndarray
    v: np.ndarray
    rows: int


class GpuBackend:
    """Per-rank compute through the C-ABI (device-resident factors)."""

    def __init__(self, store):
        from . import api
        self.api = api
        self.store = store
        self.snap = None

    def snapshot(self):
        self.snap = self.store.snapshot()
        return self.snap.total_rows

    def block(self, i):
        import ctypes as C
        from ._capi import lib
        out = C.c_void_p()
        self.api._check(lib().zsvd_snapshot_block(self.snap._h, i, C.byref(out)))
        return self.api.DeviceFactors(out.value)

    def trim(self, blk, lo, hi, trunc):
        f = self.api.trim_block(blk, lo, hi, trunc)
        return f

    def to_part(self, f, with_u=True) -> Part:
        if isinstance(f, self.api.DeviceFactors):
            f = f.download()
        return Part(f.u if with_u else None, np.asarray(f.sigma), np.asarray(f.v), f.u.shape[0])

    def stitch(self, parts: List[Part], trunc):
        fs = []
        for p in parts:
            u = p.u if p.u is not None else np.zeros((0, p.s.shape[0]))
            fs.append(self.api.SvdFactors(u, p.s, p.v))
        f = self.api.stitch(fs, trunc)
        return self.api.canonical_sign(f)

    def sign(self, f):
        return self.api.canonical_sign(f)


class NcclComm:
    """zsvd_comm: an NCCL communicator over the ranks' devices.  Rank 0 makes the
    unique id; it reaches the other ranks through ``dist`` (a
    torch.distributed-like object with broadcast_object_list)."""

    def __init__(self, rank: int, world: int, device: int, dist=None):
        import ctypes as C
        from . import api
        from ._capi import lib
        self._api, self._lib = api, lib
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            api._check(lib().zsvd_comm_unique_id(uid))
        if world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0)
            uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        api._check(lib().zsvd_comm_create(uid, world, rank, device, C.byref(h)))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self._lib().zsvd_comm_destroy(h)
            self.h = None


class ShardedStore:
    """The global stream split over ranks by contiguous block ranges."""

    def __init__(self, block_size: int, num_columns: int, rows_per_rank: int, truncation,
                 rank: int, world: int, backend_factory=None, dist=None, device: Optional[int] = None,
                 comm: Optional[NcclComm] = None):
        if rows_per_rank % block_size:
            raise ValueError("rows_per_rank must be a multiple of the block size")
        self.b, self.c = block_size, num_columns
        self.rows_per_rank = rows_per_rank
        self.rank, self.world = rank, world
        self.trunc = truncation
        self.dist = dist
        if backend_factory is None:
            from .api import BlockStore
            store = BlockStore(block_size, num_columns, policy=truncation,
                               device=rank if device is None else device)
            self.backend = GpuBackend(store)
        else:
            self.backend = backend_factory(block_size, num_columns, truncation)
        self.local_rows = 0
        self.comm = comm  # NCCL Gram exchange for the device-side sharded query

    # ---- storage: no collective
    def owner_of_row(self, row: int) -> int:
        return row // self.rows_per_rank

    def local_range(self):
        return self.rank * self.rows_per_rank, (self.rank + 1) * self.rows_per_rank

    def append_local(self, rows) -> None:
        """Appends this rank's rows (in global order of its shard)."""
        rows = np.asarray(rows, dtype=np.float64)
        if self.local_rows + rows.shape[0] > self.rows_per_rank:
            raise ValueError("shard overflow")
        self.backend.store.append(rows)
        self.local_rows += rows.shape[0]

    # ---- query: trims on owners, allgather of bands, replicated stitch
    def range_query(self, first: int, last: int):
        """Returns (u_local_rows, sigma, v, (row0, row1)) for this rank's part of [first, last]."""
        if self.comm is not None and isinstance(self.backend, GpuBackend):
            from .api import UnsupportedError
            try:
                return self._device_query(first, last)
            except UnsupportedError:
                pass  # every rank alike: gather the parts instead
        return self._band_query(first, last)

    def _device_query(self, first: int, last: int):
        import ctypes as C
        from . import api
        from ._capi import lib
        snap = self.backend.store.snapshot()
        out, off = C.c_void_p(), C.c_uint64()
        api._check(lib().zsvd_sharded_range_query(snap._h, self.comm.h, self.rows_per_rank, first, last,
                                                  self.trunc.c(), C.byref(out), C.byref(off)))
        f = api.DeviceFactors(out.value).download()
        lo = first + off.value
        return np.asarray(f.u), np.asarray(f.sigma), np.asarray(f.v), (lo, lo + f.u.shape[0])

    def _band_query(self, first: int, last: int):
        total = self._allgather(self.backend.snapshot())
        # every rank the range touches must hold all of its rows of the range
        # (shards fill independently, so a lower rank may lag): checked on all
        # ranks from the gathered totals, before any trim or collective
        rpr = self.rows_per_rank
        ok = 0 <= first <= last
        if ok:
            for r in range(first // rpr, min(last // rpr, self.world - 1) + 1):
                need_last = min(last, (r + 1) * rpr - 1)
                if r * rpr + int(total[r]) <= need_last:
                    ok = False
            ok = ok and last // rpr < self.world
        if not ok:
            from .api import RangeError
            raise RangeError("time range out of bounds")
        b = self.b
        S, E = first // b, last // b
        bpr = self.rows_per_rank // b
        owner = lambda blk: blk // bpr  # noqa: E731
        lb = lambda blk: blk - owner(blk) * bpr  # noqa: E731  (local block index)
        my_parts = []  # (global part index, Part)
        if S == E:
            if owner(S) == self.rank:
                f = self.backend.trim(self.backend.block(lb(S)), first - S * b, last - S * b, self.trunc)
                f = self.backend.sign(f)
                my_parts.append((0, self.backend.to_part(f)))
            got = self._allgather([(i, p.s, p.v) for i, p in my_parts])
            s, v = next((x[1], x[2]) for g in got for x in g)
            u = my_parts[0][1].u if my_parts else np.zeros((0, s.shape[0]))
            lo, hi = (first, last + 1) if my_parts else (first, first)
            return u, s, v, (lo, hi)
        for gi, blk in enumerate(range(S, E + 1)):
            if owner(blk) != self.rank:
                continue
            f = self.backend.block(lb(blk))
            if blk == S:
                f = self.backend.trim(f, first - S * b, b - 1, self.trunc)
            elif blk == E:
                f = self.backend.trim(f, 0, last - E * b, self.trunc)
            my_parts.append((gi, self.backend.to_part(f)))
        bands = self._allgather([(gi, p.s, p.v) for gi, p in my_parts])
        mine = dict(my_parts)
        parts = []
        for g in bands:
            for gi, s, v in g:
                parts.append((gi, mine.get(gi, Part(None, s, v, 0))))
        parts.sort(key=lambda x: x[0])
        f = self.backend.stitch([p for _, p in parts], self.trunc)
        # rows of [first, last] owned here
        lo = max(first, self.rank * self.rows_per_rank)
        hi = min(last + 1, (self.rank + 1) * self.rows_per_rank)
        if hi < lo:
            hi = lo
        return np.asarray(f.u), np.asarray(f.sigma), np.asarray(f.v), (lo, hi)

    def _allgather(self, obj):
        if self.dist is None or self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out
