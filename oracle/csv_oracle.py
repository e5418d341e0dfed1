"""CPU restatement of the reference's CSV reader (csv.hpp) — TEST
INFRASTRUCTURE ONLY: tests/ and bench.py's reference leg use it as the checker
for the GPU parser (paper_1805_00754_b200/csrc/csv_ingest.cu); the product never
imports it.

Pinned against the reference itself: tests/golden/csv_cases.json holds what the
reference's own CsvReader (compiled in place by `make -C oracle ref`) yields on
every case, and tests/test_csv_oracle.py checks this restatement against it.

Cell rule (csv.hpp:42-50, :106-112): the cell is trimmed of " \\t\\r\\f\\v";
std::from_chars (chars_format::general) must consume all of it; a value that
overflows or a non-zero value that rounds to zero is out of range, hence "not
numeric"; inf/nan parse but are "not finite".  Python's float() rounds
correctly, like from_chars, so it converts a cell once the grammar is checked.
"""
import math
import re

WS = " \t\r\f\v"
_DEC = re.compile(r"-?(?:[0-9]+(?:\.[0-9]*)?|\.[0-9]+)(?:[eE][+-]?[0-9]+)?")
_NONFIN = re.compile(r"-?(?:inf|infinity|nan|nan\([A-Za-z0-9_]*\))", re.IGNORECASE)
OK, NONFINITE, NOT_NUMERIC = 0, 1, 2


class ParseError(Exception):
    """csv ParseError (errors.hpp:34-45): message 'line N: what'."""

    def __init__(self, line, what):
        super().__init__(f"line {line}: {what}")
        self.line = line


class SchemaError(Exception):
    pass


def parse_cell(cell):
    """(kind, value) for one raw cell (csv.hpp:42-50 plus the finiteness check)."""
    c = cell.strip(WS)
    if not c:
        return NOT_NUMERIC, None
    if _NONFIN.fullmatch(c):
        return NONFINITE, None
    if not _DEC.fullmatch(c):
        return NOT_NUMERIC, None
    v = float(c)
    if math.isinf(v):
        return NOT_NUMERIC, None  # overflow: result_out_of_range
    if v == 0.0 and any(ch in "123456789" for ch in c.split("e")[0].split("E")[0]):
        return NOT_NUMERIC, None  # non-zero digits rounded to zero: underflow
    return OK, v


def read_rows(text, expected_cols=None, drop_timestamp=False):
    """Rows the reference CsvReader yields for `text` (csv.hpp:79-132), and the
    exception it raises after them (or None): (rows, exc)."""
    rows = []
    cols = 0
    saw_content = False
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline: a final newline does not start another line
    for lineno, line in enumerate(lines, start=1):
        if not line.strip(WS):
            continue
        cells = line.split(",")
        if not saw_content:
            saw_content = True
            if all(parse_cell(c)[0] == NOT_NUMERIC for c in cells):
                continue  # header
        first = 0
        if drop_timestamp:
            if len(cells) < 2:
                return rows, ParseError(lineno, "row has no value columns after the timestamp")
            first = 1
        row = []
        for c in cells[first:]:
            kind, v = parse_cell(c)
            if kind == NOT_NUMERIC:
                return rows, ParseError(lineno, f"cell '{c.strip(WS)}' is not numeric")
            if kind == NONFINITE:
                return rows, ParseError(lineno, "cell value is not finite")
            row.append(v)
        if cols == 0:
            if expected_cols is not None and len(row) != expected_cols:
                return rows, SchemaError(f"expected {expected_cols} columns, file has {len(row)}")
            cols = len(row)
        elif len(row) != cols:
            return rows, ParseError(lineno, f"expected {cols} columns, got {len(row)}")
        rows.append(row)
    return rows, None
