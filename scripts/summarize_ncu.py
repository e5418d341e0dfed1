"""Summarises ncu evidence into profiles/:
  launch list csv (gpu__time_duration, dram bytes) -> per-kernel totals and shares
  full capture (.ncu-rep)                          -> per-kernel key metrics
usage: python scripts/summarize_ncu.py <launches.csv> <full.ncu-rep|-> <out.json> [label]"""
import csv, io, json, subprocess, sys, collections

launch_csv, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
label = sys.argv[4] if len(sys.argv) > 4 else ""
rows = list(csv.reader(open(launch_csv)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
gi = h.index("Grid Size")
launch = collections.OrderedDict()
for r in rows[hdr + 1:]:
    key = r[ii]
    d = launch.setdefault(key, {"kernel": r[ki], "grid": r[gi]})
    try:
        d[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
per = collections.OrderedDict()
for d in launch.values():
    name = d["kernel"].split("(")[0]
    e = per.setdefault(name, {"launches": 0, "time_us": 0.0, "dram_bytes": 0.0})
    e["launches"] += 1
    e["time_us"] += d.get("gpu__time_duration.sum", 0.0) / 1e3
    e["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(e["time_us"] for e in per.values())
for e in per.values():
    e["share"] = e["time_us"] / tot if tot else 0.0
summary = {"label": label, "launch_list": launch_csv, "total_time_us": tot, "per_kernel": per}
if rep != "-":
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    want = {"gpu__time_duration.sum": "duration_ns", "dram__bytes_read.sum": "dram_read",
            "dram__bytes_write.sum": "dram_write", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
            "launch__registers_per_thread": "regs", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
            "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_smsp",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts"}
    idx = {n: i for i, n in enumerate(hh)}
    caps = []
    for r in rr[2:]:
        d = {"kernel": r[idx["Kernel Name"]], "grid": r[idx.get("Grid Size", 0)]}
        for m, nm in want.items():
            if m in idx:
                try:
                    d[nm] = float(r[idx[m]].replace(",", ""))
                except ValueError:
                    pass
        caps.append(d)
    summary["full_capture"] = {"report": rep, "kernels": caps}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: {kk: round(vv, 3) if isinstance(vv, float) else vv for kk, vv in v.items()} for k, v in per.items()}, indent=1))
