"""Dev probe: CSV ingest throughput on a cfg2-shaped file (b = 2000, c = 64).

Writes /tmp/zsvd_csv_cfg2.csv (rows x 64, shortest-repr doubles; cached),
then times: the GPU parse (zsvd_csv_read), ingest_csv into a fixed-rank store,
and the reference CsvReader (oracle/_ref/csv_ref, one core) on the same file.
"""
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1805_00754_b200 as z  # noqa: E402
from paper_1805_00754_b200 import api  # noqa: E402


def make(path, rows, cols=64, seed=0, rep=8):
    if os.path.exists(path):
        return
    rng = np.random.default_rng(seed)
    base = rows // rep
    a = rng.standard_normal((base, cols))
    t0 = time.time()
    body = "\n".join(",".join(map(repr, r)) for r in a.tolist()) + "\n"
    with open(path, "w") as f:
        for _ in range(rep):
            f.write(body)
    print(f"wrote {path}: {os.path.getsize(path) / 1e9:.2f} GB in {time.time() - t0:.1f}s", flush=True)


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    path = f"/tmp/zsvd_csv_cfg2_{rows}.csv"
    make(path, rows)
    size = os.path.getsize(path)
    for i in range(4):
        t0 = time.perf_counter()
        f = api._CsvFile(path, None)
        t1 = time.perf_counter()
        print(f"parse {i}: {t1 - t0:.3f}s  {size / (t1 - t0) / 1e9:.2f} GB/s  {f.rows / (t1 - t0):.3e} rows/s "
              f"rows={f.rows} cols={f.cols}", flush=True)
        del f
    for i in range(3):
        t0 = time.perf_counter()
        st = z.ingest_csv(path, 2000, policy=z.Truncation.fixed_rank(20))
        st.sync()
        t1 = time.perf_counter()
        print(f"ingest {i}: {t1 - t0:.3f}s  {st.total_rows() / (t1 - t0):.3e} rows/s sealed={st.sealed_count()}",
              flush=True)
        del st
    ref = os.path.join(ROOT, "oracle", "_ref", "csv_ref")
    if os.path.exists(ref) and len(sys.argv) > 2:
        out = subprocess.run([ref, path, "-1", "0", "T"], capture_output=True, text=True).stdout
        n, s = out.split()[1:3]
        print(f"reference CsvReader: {float(s):.2f}s  {int(n) / float(s):.3e} rows/s  {size / float(s) / 1e9:.3f} GB/s")


if __name__ == "__main__":
    main()
