"""profiles/ncu_summary.json from this round's ncu artefacts in gpurun_out/ (dev tool):
the serialised launch list of one 500-block cfg2 flush + 3 queries, and the
full-capture digests (scripts/ncu_brief.py)."""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01m"
lc = os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
rows = list(csv.reader(open(lc)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]
ki, mi, vi, ii, gi = (H.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
L, order = {}, []
for r in rows[h + 1:]:
    if r[ii] not in L:
        order.append(r[ii])
    d = L.setdefault(r[ii], {"k": r[ki].split("(")[0], "g": r[gi]})
    d[r[mi]] = float(r[vi].replace(",", ""))
launches = [L[i] for i in order]
byte = lambda d: d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
stor = [d for d in launches if ", 500, 1)" in d["g"]] + [next(d for d in launches if d["k"] == "svd_fallback_kernel")]
tot = sum(d["gpu__time_duration.sum"] for d in stor) / 1e3
q = launches[-10:]
briefs = []
for rep in (f"{tag}_storage_m2", f"{tag}_storage_p3", f"{tag}_trim_qr"):
    p = os.path.join(ROOT, "gpurun_out", rep + ".ncu-rep")
    if os.path.exists(p):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_brief.py"), p], capture_output=True, text=True).stdout
        briefs += [f"== {rep}"] + out.strip().split("\n")
summary = {
    "round": tag,
    "storage_flush_cfg2_500": {
        "source": f"profiles/{tag}_launches_storage500_query.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  "dram__bytes_write.sum --clock-control none, ZSVD_DEV_LANES=1: one 500-block flush, serialised, cold caches)",
        "time_us": tot, "dram_bytes_per_launch": sum(byte(d) for d in stor), "algorithmic_bytes_per_launch": 677200000.0,
        "kernels": {d["k"]: {"grid": d["g"], "time_us": d["gpu__time_duration.sum"] / 1e3, "dram_bytes": byte(d),
                             "share_of_flush": d["gpu__time_duration.sum"] / 1e3 / tot} for d in stor}},
    "query_cfg2_L320000": {"source": "same launch list, last of 3 queries",
                           "time_us": sum(d["gpu__time_duration.sum"] for d in q) / 1e3,
                           "kernels": [{"kernel": d["k"], "grid": d["g"], "time_us": d["gpu__time_duration.sum"] / 1e3} for d in q]},
    "full_captures": {"note": "ncu --set full --clock-control none; digests by scripts/ncu_brief.py", "digest": briefs},
}
json.dump(summary, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps({"flush_us": tot, "flush_dram": summary["storage_flush_cfg2_500"]["dram_bytes_per_launch"],
                  "query_us": summary["query_cfg2_L320000"]["time_us"]}))
