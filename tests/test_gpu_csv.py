"""CSV ingestion on the GPU (csv.hpp): the device parser
against the reference's own CsvReader (golden cases), against the oracle
restatement on randomized files, on multi-chunk files (tiny chunks force every
boundary case), and ingestion into a store (cmd_ingest, commands.hpp:106-139)."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_1805_00754_b200 as z

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import csv_oracle as CO  # noqa: E402
import oracle as O  # noqa: E402
from parity import assert_parity  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "csv_cases.json")))["cases"]


def write(path, text):
    with open(path, "wb") as f:
        f.write(text.encode("latin-1"))
    return str(path)


def read_all(path, expected=None, drop=False):
    """Rows a CsvReader yields and the exception it ends with (or None)."""
    rdr = z.CsvReader(path, z.CsvOptions(expected, drop))
    rows = []
    try:
        while True:
            r = rdr.next()
            if r is None:
                return rows, None
            rows.append(r.copy())
    except (z.ParseError, z.SchemaError) as e:
        return rows, e


def as_bits(rows):
    return [[struct.unpack(">Q", struct.pack(">d", float(v)))[0] for v in r] for r in rows]


def same_as_oracle(rows, exc, o_rows, o_exc):
    assert as_bits(rows) == as_bits(o_rows)
    if o_exc is None:
        assert exc is None
    else:
        assert type(exc).__name__ == type(o_exc).__name__ and str(exc) == str(o_exc)
        if isinstance(o_exc, CO.ParseError):
            assert exc.line == o_exc.line


@pytest.mark.parametrize("case", GOLDEN, ids=lambda c: c["name"])
def test_golden_cases_match_reference_reader(tmp_path, case):
    p = write(tmp_path / "c.csv", case["text"])
    rows, exc = read_all(p, case["expected_cols"], case["drop_timestamp"])
    assert as_bits(rows) == [[int(h, 16) for h in r] for r in case["rows"]]
    e = case["error"]
    if e is None:
        assert exc is None
    else:
        assert type(exc).__name__ == e["type"] and str(exc) == e["what"]
        if e["type"] == "ParseError":
            assert exc.line == e["line"]


def test_reader_api(tmp_path):
    # io_test.cpp:127-135 and read_csv_rows / read_csv_matrix (csv.hpp:153-177)
    with pytest.raises(z.IoError):
        z.CsvReader("/nonexistent/really_not_here.csv")
    p = write(tmp_path / "e.csv", "")
    assert z.read_csv_rows(p) == []
    with pytest.raises(z.InvalidInputError):
        z.read_csv_matrix(p)
    p = write(tmp_path / "m.csv", "a,b\n1,2\n3,4\n")
    r = z.CsvReader(p)
    assert r.cols() == 0
    assert list(r.next()) == [1.0, 2.0] and r.cols() == 2
    assert np.array_equal(z.read_csv_matrix(p), [[1, 2], [3, 4]])
    with pytest.raises(z.ParseError) as ei:
        z.read_csv_rows(write(tmp_path / "r.csv", "1,2\n3,4,5\n"))
    assert ei.value.line == 2


CELLS = [
    lambda r: "%.17g" % r.uniform(-1, 1),
    lambda r: repr(struct.unpack("<d", struct.pack("<Q", r.getrandbits(63)))[0]),
    lambda r: "%.6e" % (r.uniform(-1e6, 1e6)),
    lambda r: str(r.randint(-10 ** 20, 10 ** 20)),
    lambda r: "%d.%de%d" % (r.randint(0, 999), r.randint(0, 10 ** 9), r.randint(-330, 310)),
    lambda r: " %.17g\t" % r.uniform(-1e-300, 1e-300),
    lambda r: "0." + "".join(r.choice("0123456789") for _ in range(r.randint(20, 60))),
]


def random_text(seed, rows, cols, blank_every=0, header=False, crlf=False):
    import random
    r = random.Random(seed)
    lines = ["t" + ",t".join(str(i) for i in range(cols))] if header else []
    for i in range(rows):
        lines.append(",".join(CELLS[r.randrange(len(CELLS))](r) for _ in range(cols)))
        if blank_every and i % blank_every == 3:
            lines.append(" \t")
    return ("\r\n" if crlf else "\n").join(lines) + ("\r\n" if crlf else "\n")


@pytest.mark.parametrize("seed,rows,cols,blank,header,crlf", [(1, 400, 7, 0, False, False),
                                                              (2, 300, 33, 11, True, True),
                                                              (3, 50, 300, 4, True, False)])
def test_random_files_match_oracle(tmp_path, seed, rows, cols, blank, header, crlf):
    text = random_text(seed, rows, cols, blank, header, crlf)
    rows_g, exc = read_all(write(tmp_path / "r.csv", text))
    same_as_oracle(rows_g, exc, *CO.read_rows(text))


def test_round_trip_of_17g_matrix(tmp_path):
    """A %.17g matrix (the reference tests' write_csv format) parses back to the
    same doubles bit for bit (size-independent property)."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((20000, 64)) * np.logspace(-3, 3, 64)
    p = tmp_path / "m.csv"
    np.savetxt(p, a, fmt="%.17g", delimiter=",")
    got = z.read_csv_matrix(str(p))
    assert got.shape == a.shape and np.array_equal(got.view(np.uint64), a.view(np.uint64))


SMALL_CHUNK_SCRIPT = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
sys.path.insert(0, os.path.join(sys.argv[1], "oracle"))
import test_gpu_csv as T, csv_oracle as CO
tmp = sys.argv[2]
for i, case in enumerate(T.GOLDEN):
    p = T.write(os.path.join(tmp, "g%d.csv" % i), case["text"])
    rows, exc = T.read_all(p, case["expected_cols"], case["drop_timestamp"])
    o_rows, o_exc = CO.read_rows(case["text"], case["expected_cols"], case["drop_timestamp"])
    T.same_as_oracle(rows, exc, o_rows, o_exc)
for seed in range(4):
    text = T.random_text(100 + seed, 300, 9, blank_every=5 + seed, header=seed % 2 == 0, crlf=seed == 3)
    if seed == 1:
        lines = text.split("\n"); lines[211] = lines[211] + ",9"; text = "\n".join(lines)
    if seed == 2:
        lines = text.split("\n"); lines[150] = "1,x," + lines[150]; text = "\n".join(lines)
    p = T.write(os.path.join(tmp, "r%d.csv" % seed), text)
    T.same_as_oracle(*T.read_all(p), *CO.read_rows(text))
# a line far longer than a chunk (buffer growth) and a header split across chunks
long_text = "h" * 5000 + ",x\n" + ",".join(["1.25"] * 3000) + "\n" + ",".join(["2.5"] * 3000)
p = T.write(os.path.join(tmp, "long.csv"), long_text)
T.same_as_oracle(*T.read_all(p), *CO.read_rows(long_text))
print("SMALL-CHUNK-OK")
"""


def test_tiny_chunks_everywhere(tmp_path):
    """Chunks of 256 bytes: headers, blank lines, errors and long lines across
    chunk boundaries, carries and pinned-buffer growth."""
    env = dict(os.environ, ZSVD_CSV_CHUNK_BYTES="256")
    out = subprocess.run([sys.executable, "-c", SMALL_CHUNK_SCRIPT, ROOT, str(tmp_path)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert "SMALL-CHUNK-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]


def test_multi_chunk_file_with_late_error(tmp_path):
    """A ~40 MB file (two 32 MB chunks): blank lines, then a ragged row deep in the
    second chunk; the rows before it are yielded, the line number is exact."""
    rng = np.random.default_rng(9)
    a = rng.uniform(-1, 1, (240000, 8))
    body = "\n".join(",".join("%.17g" % v for v in row) for row in a[:1000]) + "\n"
    blocks = [body] * 240
    text = "c0,c1,c2,c3,c4,c5,c6,c7\n\n" + "".join(blocks)
    lines = text.split("\n")
    bad = 230000
    lines[bad] = lines[bad] + ",1"
    text = "\n".join(lines)
    p = write(tmp_path / "big.csv", text)
    assert os.path.getsize(p) > 33 << 20
    rows, exc = read_all(p)
    assert isinstance(exc, z.ParseError) and exc.line == bad + 1
    assert str(exc) == f"line {bad + 1}: expected 8 columns, got 9"
    assert len(rows) == bad - 2
    tiled = np.tile(a[:1000], (240, 1))
    assert np.array_equal(np.array(rows[:5000]), tiled[:5000]) and np.array_equal(np.array(rows[-10:]),
                                                                                   tiled[bad - 12:bad - 2])


def test_ingest_matches_direct_store(tmp_path):
    """cmd_ingest core: store from the CSV == store from the same rows appended
    directly (bitwise); commands_test ReportsSealedBlockCount (3000 x 4, b 1000)."""
    rng = np.random.default_rng(401)
    raw = rng.uniform(-1, 1, (3000, 4))
    p = tmp_path / "in.csv"
    np.savetxt(p, raw, fmt="%.17g", delimiter=",")
    st = z.ingest_csv(str(p), 1000, 0.98)
    assert st.total_rows() == 3000 and st.sealed_count() == 3
    ref = z.BlockStore(1000, 4, 0.98)
    ref.append(raw)
    for i in range(3):
        f, g = st.block(i), ref.block(i)
        assert np.array_equal(f.sigma, g.sigma) and np.array_equal(f.u, g.u)
    o = O.Store(1000, 4, 0.98)
    o.append(raw)
    assert_parity(st.block(1), o.block(1), what="ingested block 1")
    with pytest.raises(z.InvalidInputError):
        z.ingest_csv(write(tmp_path / "e.csv", ""), 10, 0.98)
    with pytest.raises(z.InvalidParameterError):
        z.ingest_csv(str(p), 0, 0.98)
    with pytest.raises(z.InvalidParameterError):
        z.ingest_csv(str(p), 10, 1.5)


def test_append_csv_is_atomic(tmp_path):
    rng = np.random.default_rng(3)
    raw = rng.standard_normal((500, 6))
    st = z.BlockStore(64, 6, policy=z.Truncation.fixed_rank(3))
    st.append(raw[:100])
    good = tmp_path / "good.csv"
    np.savetxt(good, raw[100:], fmt="%.17g", delimiter=",")
    text = open(good).read().split("\n")
    text[250] = text[250].replace(",", ",nan,", 1)
    bad = write(tmp_path / "bad.csv", "\n".join(text))
    with pytest.raises(z.ParseError) as ei:
        st.append_csv(bad)
    assert ei.value.line == 251 and st.total_rows() == 100
    with pytest.raises(z.InvalidInputError):
        st.append_csv(write(tmp_path / "w.csv", "1,2,3\n"))
    assert st.append_csv(str(good)) == 400 and st.total_rows() == 500
    ref = z.BlockStore(64, 6, policy=z.Truncation.fixed_rank(3))
    ref.append(raw)
    for i in range(st.sealed_count()):
        assert np.array_equal(st.block(i).sigma, ref.block(i).sigma)
