"""Generates tests/golden/csv_cases.json: CSV inputs and what the reference's own
CsvReader (csv.hpp, compiled in place by `make -C oracle ref` into
oracle/_ref/csv_ref) yields for each — rows as IEEE bit patterns, then the
exception type, line and message, if any.  Run in the build container (it needs
/root/reference); the JSON is committed and read by tests on any machine.

The first cases are the reference's own io_test CsvReader inputs
(tests/io_test.cpp:52-135); the rest probe the edges of the same rules."""
import json
import os
import random
import struct
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "csv_ref")


def halfway(x):
    """Exact decimal text of the midpoint between x > 0 and its successor."""
    m, e = __import__("math").frexp(x)
    mi = int(m * (1 << 53))
    e -= 53
    H, t = 2 * mi + 1, e - 1
    if t >= 0:
        return str(H << t)
    digits = str(H * 5 ** (-t))
    frac = -t
    if frac >= len(digits):
        return "0." + "0" * (frac - len(digits)) + digits
    return digits[:-frac] + "." + digits[-frac:]


def cases():
    c = [
        # tests/io_test.cpp:52-135
        ("io_plain_rows", "1,2\n3,4\n5,6\n", None, False),
        ("io_header", "a,b\n1,2\n", None, False),
        ("io_non_numeric_cell", "1,x\n", None, False),
        ("io_ragged_row", "1,2\n3,4,5\n", None, False),
        ("io_expected_cols_schema", "1,2,3\n", 2, False),
        ("io_drop_timestamp", "time,s1,s2\n100,1.5,2.5\n200,3.5,4.5\n", None, True),
        ("io_scientific_whitespace", "  1.5e2 , -3E-1 \n 2 , 0.25 \n", None, False),
        ("io_non_finite", "1,2\n3,inf\n", None, False),
        ("io_empty_file", "", None, False),
        # edges of the same rules
        ("blank_lines_and_crlf", "\n  \n1,2\r\n\r\n3,4\r\n\t\n", None, False),
        ("no_trailing_newline", "1,2\n3,4", None, False),
        ("header_only", "x,y,z\n", None, False),
        ("header_after_blank_lines", "\n\n a , b \n1,2\n", None, False),
        ("second_line_textual_is_error", "1,2\na,b\n", None, False),
        ("partly_numeric_first_line_is_data", "1,b\n2,3\n", None, False),
        ("header_with_inf_is_data", "inf,nan\n1,2\n", None, False),
        ("trailing_comma", "1,2,\n", None, False),
        ("empty_cell", "1,,2\n", None, False),
        ("whitespace_cell", "1, \t ,2\n", None, False),
        ("fewer_columns", "1,2,3\n4,5\n", None, False),
        ("bad_cell_beats_ragged", "1,2\n3,x,5\n", None, False),
        ("bad_cell_in_first_row_beats_schema", "1,x,3\n", 2, False),
        ("schema_ok", "1,2\n3,4\n", 2, False),
        ("drop_ts_single_column", "1,2\n5\n", None, True),
        ("drop_ts_textual_stamp", "2020-01-01,1,2\n2020-01-02,3,4\n", None, True),
        ("drop_ts_header", "t,a\n1,2\n", None, True),
        ("drop_ts_schema", "0,1,2\n", 3, True),
        ("nan_forms", "nan(abc_1),1\n", None, False),
        ("nan_bad_forms", "nan(a-b),1\n", None, False),
        ("infinity_word", "1,-Infinity\n", None, False),
        ("plus_sign_not_numeric", "1,+2\n", None, False),
        ("hex_not_numeric", "0x10,1\n", None, False),
        ("underscore_not_numeric", "1_0,1\n", None, False),
        ("exponent_without_digits", "1e,2\n", None, False),
        ("leading_dot_trailing_dot", ".5,5.,-.25,-0,0.\n", None, False),
        ("overflow_not_numeric", "1,1e309\n", None, False),
        ("max_double", "1.7976931348623157e308,-1.7976931348623158e308\n", None, False),
        ("just_over_max", "1,1.7976931348623159e308\n", None, False),
        ("underflow_not_numeric", "1,1e-400\n", None, False),
        ("zero_with_huge_exponent", "0e99999999999999999999,-0.000e-9999\n", None, False),
        ("subnormals", "4.9406564584124654e-324,2.4703282292062328e-324,2.2250738585072009e-308,1e-310\n", None, False),
        ("below_half_min_subnormal", "1,2.4703282292062327e-324\n", None, False),
        ("single_bad_cell_is_header", "1e-400\n2\n", None, False),
        ("integers_near_2_53", "9007199254740993,9007199254740995,18446744073709551615,123456789012345678901234567890\n", None, False),
        ("long_mantissas", "0." + "3" * 400 + ",1" + "0" * 300 + "e-300," + "9" * 30 + "e-20\n", None, False),
        ("tabs_and_formfeeds", "\f1\v,\t2 \n", None, False),
        ("many_columns", ",".join(str(i * 0.5) for i in range(300)) + "\n" + ",".join(str(-i) for i in range(300)) + "\n", None, False),
    ]
    rng = random.Random(20180502)
    hw = []
    for _ in range(24):
        x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(62) | (1 << 52)))[0]
        h = halfway(x)
        hw.append(h)
        hw.append(h[:40] if len(h) > 40 else h)
        hw.append(h + "0000001")
    for i in range(0, len(hw), 6):
        c.append((f"halfway_points_{i // 6}", ",".join(hw[i:i + 6]) + "\n", None, False))
    # a random %.17g matrix (the reference tests' write_csv format, commands_test.cpp:21-34)
    lines = []
    for _ in range(40):
        lines.append(",".join("%.17g" % rng.uniform(-1, 1) for _ in range(7)))
    c.append(("random_17g_matrix", "\n".join(lines) + "\n", None, False))
    lines = []
    for _ in range(40):
        lines.append(",".join(repr(struct.unpack("<d", struct.pack("<Q", rng.getrandbits(63)))[0]) for _ in range(5)))
    c.append(("random_bit_patterns", "\n".join(lines) + "\n", None, False))
    return c


def run(text, expected, drop):
    with tempfile.NamedTemporaryFile("wb", suffix=".csv", delete=False) as f:
        f.write(text.encode("latin-1"))
        path = f.name
    try:
        out = subprocess.run([REF, path, str(-1 if expected is None else expected), "1" if drop else "0"],
                             check=True, capture_output=True).stdout.decode("latin-1")
    finally:
        os.unlink(path)
    rows, err = [], None
    for line in out.splitlines():
        if line.startswith("R"):
            rows.append(line.split()[1:])
        elif line.startswith("E "):
            _, typ, ln, what = line.split(" ", 3)
            err = {"type": typ, "line": int(ln), "what": what}
    return rows, err


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    out = []
    for name, text, expected, drop in cases():
        rows, err = run(text, expected, drop)
        out.append({"name": name, "text": text, "expected_cols": expected, "drop_timestamp": drop,
                    "rows": rows, "error": err})
    path = os.path.join(ROOT, "tests", "golden", "csv_cases.json")
    with open(path, "w") as f:
        json.dump({"generator": "scripts/gen_csv_golden.py via oracle/_ref/csv_ref (reference csv.hpp)",
                   "cases": out}, f, indent=1)
    print(f"{len(out)} cases -> {path}")


if __name__ == "__main__":
    main()
