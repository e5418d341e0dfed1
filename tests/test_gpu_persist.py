"""ZSVD v1 persistence (serialize.hpp): the reference's
io_test SaveLoad cases on the GPU store, resume-after-load, and format
compatibility both ways with a writer/reader of the reference layout fed by
the oracle."""
import os
import struct

import numpy as np
import pytest

import oracle as O
import paper_1805_00754_b200 as z
from parity import assert_parity

pytestmark = pytest.mark.gpu
HEADER = 4 + 4 + 4 + 4 + 8 + 8 + 8 + 1  # serialize.hpp:144


def store_from(raw, b, xi):
    st = z.BlockStore(b, raw.shape[1], xi)
    st.append(raw)
    return st


def blocks(st):
    n = st.sealed_count() + (1 if st.info().open_rows else 0)
    return [st.block(i) for i in range(n)]


def bitwise_equal(f, g):
    return (np.array_equal(f.u, g.u) and np.array_equal(f.sigma, g.sigma) and np.array_equal(f.v, g.v))


# ---- the reference layout, written / read in Python (serialize.hpp:3-11) ----
def write_ref_file(path, b, c, xi, total, sealed, open_block):
    buf = bytearray(b"ZSVD")
    buf += struct.pack("<IIIdQQ", 1, b, c, xi, len(sealed), total)
    buf += b"\x01" if open_block is not None else b"\x00"
    def fac(f):
        out = struct.pack("<I", f.rank)
        out += np.ascontiguousarray(f.u, dtype="<f8").tobytes()
        out += np.ascontiguousarray(f.s, dtype="<f8").tobytes()
        out += np.ascontiguousarray(f.v, dtype="<f8").tobytes()
        return out
    for i, f in enumerate(sealed):
        buf += struct.pack("<Q", i) + fac(f)
    if open_block is not None:
        rows, f = open_block
        buf += struct.pack("<QQ", len(sealed), rows) + fac(f)
    open(path, "wb").write(bytes(buf))


def read_ref_file(path):
    data = open(path, "rb").read()
    assert data[:4] == b"ZSVD"
    ver, b, c, xi, ns, total = struct.unpack_from("<IIIdQQ", data, 4)
    pos = HEADER
    has_open = data[pos - 1]
    def fac(rows):
        nonlocal pos
        (k,) = struct.unpack_from("<I", data, pos)
        pos += 4
        u = np.frombuffer(data, "<f8", rows * k, pos).reshape(rows, k)
        pos += 8 * rows * k
        s = np.frombuffer(data, "<f8", k, pos)
        pos += 8 * k
        v = np.frombuffer(data, "<f8", c * k, pos).reshape(c, k)
        pos += 8 * c * k
        return u, s, v
    out = []
    for i in range(ns):
        (idx,) = struct.unpack_from("<Q", data, pos)
        pos += 8
        assert idx == i
        out.append(fac(b))
    if has_open:
        idx, rows = struct.unpack_from("<QQ", data, pos)
        pos += 16
        out.append(fac(rows))
    assert pos == len(data)
    return (b, c, xi, total), out


def test_round_trip_preserves_everything(tmp_path):
    rng = np.random.default_rng(211)
    st = store_from(rng.uniform(-1, 1, (22, 4)), 5, 0.95)
    assert st.sealed_count() == 4 and st.info().open_rows == 2
    p = tmp_path / "rt.zsvd"
    z.save_store(st, p)
    ld = z.load_store(p)
    assert (ld.block_size(), ld.num_columns(), ld.energy_threshold(), ld.total_rows()) == (5, 4, 0.95, 22)
    assert ld.sealed_count() == 4 and ld.info().open_rows == 2
    for f, g in zip(blocks(st), blocks(ld)):
        assert bitwise_equal(f, g)
    # a save of the loaded store is the same file, byte for byte
    p2 = tmp_path / "rt2.zsvd"
    z.save_store(ld, p2)
    assert open(p, "rb").read() == open(p2, "rb").read()


def test_saving_twice_is_byte_identical_and_sizes(tmp_path):
    rng = np.random.default_rng(227)
    st = store_from(rng.uniform(-1, 1, (17, 4)), 5, 0.9)
    a, b = tmp_path / "a", tmp_path / "b"
    z.save_store(st, a)
    z.save_store(st, b)
    assert open(a, "rb").read() == open(b, "rb").read()
    expected = HEADER + sum(8 + 4 + f.rank() * (5 + 1 + 4) * 8 for f in blocks(st)[:3])
    expected += 8 + 8 + 4 + blocks(st)[3].rank() * (2 + 1 + 4) * 8
    assert os.path.getsize(a) == expected


def test_empty_store_is_header_only(tmp_path):
    st = z.BlockStore(8, 3, 0.98)
    p = tmp_path / "e"
    z.save_store(st, p)
    assert os.path.getsize(p) == HEADER
    ld = z.load_store(p)
    assert ld.total_rows() == 0 and ld.sealed_count() == 0


def _saved(tmp_path, raw, b, xi, name):
    st = store_from(raw, b, xi)
    p = tmp_path / name
    z.save_store(st, p)
    return p, bytearray(open(p, "rb").read())


def test_damaged_files(tmp_path):
    rng = np.random.default_rng(229)
    p, data = _saved(tmp_path, rng.uniform(-1, 1, (8, 3)), 4, 1.0, "m")
    bad = bytearray(data)
    bad[0] = ord("X")
    open(p, "wb").write(bad)
    with pytest.raises(z.FormatError):
        z.load_store(p)
    bad = bytearray(data)
    bad[4] = 7
    open(p, "wb").write(bad)
    with pytest.raises(z.FormatError):
        z.load_store(p)
    open(p, "wb").write(data[: len(data) // 2])
    with pytest.raises(z.CorruptionError):
        z.load_store(p)
    open(p, "wb").write(data + b"extra")
    with pytest.raises(z.CorruptionError):
        z.load_store(p)
    # header claims two sealed blocks, the payload holds one
    p1, d1 = _saved(tmp_path, rng.uniform(-1, 1, (4, 3)), 4, 1.0, "c")
    d1[24] = 2
    open(p1, "wb").write(d1)
    with pytest.raises(z.CorruptionError):
        z.load_store(p1)
    # smash the exponent byte of the first U entry (past index u64 + k u32)
    p2, d2 = _saved(tmp_path, rng.uniform(-1, 1, (4, 3)), 4, 1.0, "i")
    d2[HEADER + 12 + 7] = 0x7F
    open(p2, "wb").write(d2)
    with pytest.raises(z.CorruptionError):
        z.load_store(p2)
    with pytest.raises(z.IoError):
        z.load_store(tmp_path / "missing")


def test_fixed_rank_store_round_trip(tmp_path):
    """FIXED_RANK stores (the BASELINE configs) save as the version-2 extension:
    the v1 layout plus the rank after the threshold field.  They load back with
    their policy, factors bit for bit, and keep appending like the original."""
    rng = np.random.default_rng(23)
    b, c, k = 50, 8, 3
    raw = rng.standard_normal((5 * b + 17, c)) @ np.diag(np.linspace(4, 0.5, c))
    st = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
    st.append(raw[: 3 * b + 9])
    p = tmp_path / "fixed"
    z.save_store(st, p)
    data = open(p, "rb").read()
    assert data[:4] == b"ZSVD" and int.from_bytes(data[4:8], "little") == 2
    assert int.from_bytes(data[24:32], "little") == k
    ld = z.load_store(p)
    assert ld.truncation.policy == z.Truncation.fixed_rank(k).policy and ld.truncation.k == k
    for f, g in zip(blocks(st), blocks(ld)):
        assert np.array_equal(f.u, g.u) and np.array_equal(f.sigma, g.sigma) and np.array_equal(f.v, g.v)
    ld.append(raw[3 * b + 9:])
    st.append(raw[3 * b + 9:])
    for i in range(3, 5):
        assert_parity(ld.block(i), st.block(i), what=f"resumed fixed-rank block {i}")
    # a re-save is byte-identical
    q = tmp_path / "fixed2"
    z.save_store(z.load_store(p), q)
    assert open(q, "rb").read() == data


def test_truncated_counts_fail_before_allocation(tmp_path):
    """A header claiming far more blocks than the file holds is CorruptionError
    ('store file is truncated', serialize.hpp:68-71), not an allocation failure."""
    rng = np.random.default_rng(3)
    p, d = _saved(tmp_path, rng.uniform(-1, 1, (9, 3)), 4, 1.0, "t")
    d[24:32] = (10 ** 12).to_bytes(8, "little")  # sealed count
    open(p, "wb").write(d)
    with pytest.raises(z.CorruptionError, match="truncated"):
        z.load_store(p)


def test_resume_after_load_matches_uninterrupted_store(tmp_path):
    rng = np.random.default_rng(5)
    b, c = 40, 6
    raw = rng.standard_normal((7 * b + 13, c)) @ np.diag(np.linspace(3, 0.5, c))
    cut = 3 * b + 17  # inside a block: the open block is resumed from its factors
    st = store_from(raw[:cut], b, 0.97)
    p = tmp_path / "r"
    z.save_store(st, p)
    ld = z.load_store(p)
    ld.append(raw[cut:])
    ref = O.Store(b, c, 0.97)
    ref.append(raw)
    assert ld.sealed_count() == 7 and ld.total_rows() == raw.shape[0]
    for i in range(8):
        assert_parity(ld.block(i), ref.block(i), what=f"resumed block {i}")
    for a0, a1 in [(0, raw.shape[0] - 1), (100, 250), (cut - 5, cut + 60)]:
        assert_parity(z.range_query(ld, a0, a1).factors, ref.range_query(a0, a1), what=f"[{a0},{a1}]")


def test_reference_layout_both_ways(tmp_path):
    """A file written in the reference layout from oracle factors loads into the
    GPU store bit for bit; a file the GPU store writes parses in that layout."""
    rng = np.random.default_rng(17)
    b, c = 30, 5
    raw = rng.standard_normal((4 * b + 11, c))
    ref = O.Store(b, c, 0.9)
    ref.append(raw)
    sealed = [ref.block(i) for i in range(ref.sealed_count)]
    open_f = ref.block(ref.sealed_count)
    p = tmp_path / "from_oracle"
    write_ref_file(p, b, c, 0.9, raw.shape[0], sealed, (ref.open_rows, open_f))
    ld = z.load_store(p)
    for f, g in zip(sealed + [open_f], blocks(ld)):
        assert np.array_equal(f.u, g.u) and np.array_equal(f.s, g.sigma) and np.array_equal(f.v, g.v)
    for a0, a1 in [(3, 70), (0, raw.shape[0] - 1)]:
        assert_parity(z.range_query(ld, a0, a1).factors, ref.range_query(a0, a1), what=f"loaded [{a0},{a1}]")
    st = store_from(raw, b, 0.9)
    q = tmp_path / "from_gpu"
    z.save_store(st, q)
    (hb, hc, hxi, total), fs = read_ref_file(q)
    assert (hb, hc, hxi, total) == (b, c, 0.9, raw.shape[0])
    for (u, s, v), g in zip(fs, blocks(st)):
        assert np.array_equal(u, g.u) and np.array_equal(s, g.sigma) and np.array_equal(v, g.v)


@pytest.mark.gpu
def test_store_from_parts_round_trip():
    """BlockStore::from_parts (store.hpp:206-231): a store rebuilt from another's
    sealed and open factors answers every query bit for bit like it; counts or
    shapes that do not fit raise InvalidInputError (store_test.cpp:262-273)."""
    rng = np.random.default_rng(7)
    b, c, k = 50, 8, 4
    raw = rng.standard_normal((4 * b + 17, c))
    a = z.BlockStore(b, c, policy=z.Truncation.fixed_rank(k))
    a.append(raw)
    sealed = [a.block(i) for i in range(a.sealed_count())]
    open_f = a.block(a.sealed_count())
    r = z.store_from_parts(b, c, z.Truncation.fixed_rank(k), sealed, (a.open_rows(), open_f))
    assert r.sealed_count() == a.sealed_count() and r.total_rows() == a.total_rows()
    for i in range(a.sealed_count() + 1):
        fa, fr = a.block(i), r.block(i)
        assert np.array_equal(fa.u, fr.u) and np.array_equal(fa.sigma, fr.sigma) and np.array_equal(fa.v, fr.v)
    for first, last in [(0, raw.shape[0] - 1), (13, 3 * b + 2), (4 * b + 1, raw.shape[0] - 1)]:
        qa = z.range_query(a, first, last).factors
        qr = z.range_query(r, first, last).factors
        assert np.array_equal(qa.u, qr.u) and np.array_equal(qa.sigma, qr.sigma), (first, last)
    with pytest.raises(z.InvalidInputError):  # open block longer than a block
        z.store_from_parts(b, c, z.Truncation.fixed_rank(k), sealed, (b + 1, sealed[0]))
    with pytest.raises(z.InvalidInputError):
        z.store_from_parts(b + 1, c, z.Truncation.fixed_rank(k), sealed, None)  # wrong block rows
