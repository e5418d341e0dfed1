"""One-line-per-kernel digest of an ncu report: time, grid, pipe / memory
utilisation and the top stall reasons.  python scripts/ncu_brief.py rep.ncu-rep"""
import csv, io, subprocess, sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
h = r[0]
keys = {"time_us": "gpu__time_duration.sum", "grid": "launch__grid_size", "regs": "launch__registers_per_thread",
        "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "fp64%": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smem%": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active"}
for v in r[2:]:
    d = dict(zip(h, v))
    parts = [d.get("Kernel Name", "?")[:48]]
    for k, m in keys.items():
        parts.append(f"{k}={d.get(m, 'na')}")
    print(" ".join(parts))
    st = []
    for n, x in d.items():
        if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued"):
            try:
                st.append((float(x.replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(a for a, _ in st) or 1
    print("    stalls:", ", ".join(f"{n} {100 * a / tot:.0f}%" for a, n in sorted(st)[-7:][::-1]))
