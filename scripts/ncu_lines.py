"""Attribute ncu SASS-level stall samples to source lines (when ncu cannot
import the sources): joins `ncu --page source --print-source sass` with the
line table of `nvdisasm -g` on the same cubin.

  python scripts/ncu_lines.py <report.ncu-rep> <mangled kernel> [top]
"""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_1805_00754_b200", "libzsvd.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
lines = {}
cur_line = None
inside = False
for ln in sass.splitlines():
    if ln.startswith(".text.") and ln.rstrip(":").endswith(kern):
        inside = True
        continue
    if inside and ln.startswith("//---------------------"):
        break
    if not inside:
        continue
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:
        cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_line is not None:
        lines[int(m.group(1), 16)] = cur_line
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
funcs = {}
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = r[1]
        funcs[cur] = []
    elif cur is not None:
        funcs[cur].append(r)
sub_tot = {}
main = None
for name, rs in funcs.items():
    h = rs[0]
    wi = h.index("Warp Stall Sampling (All Samples)")
    t = 0
    for r in rs[1:]:
        try:
            t += int(r[wi])
        except (ValueError, IndexError):
            pass
    sub_tot[name] = t
    if main is None or t > sub_tot[main]:
        main = name
print("per function samples:", {k[:50]: v for k, v in sub_tot.items() if v})
rs = funcs[main]
h = rs[0]
ai, wi = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rs[1:] if len(r) > wi]
base = int(data[0][ai], 16)
acc = collections.Counter()
tot = 0
for r in data:
    try:
        s = int(r[wi])
    except ValueError:
        continue
    off = int(r[ai], 16) - base
    acc[lines.get(off, ("?", -1))] += s
    tot += s
srcs = {}
def text_of(f, line):
    path = os.path.join(ROOT, "paper_1805_00754_b200", "csrc", f)
    if f not in srcs:
        srcs[f] = open(path).read().splitlines() if os.path.exists(path) else []
    src = srcs[f]
    return src[line - 1].strip()[:90] if 0 < line <= len(src) else "?"
print("total samples", tot)
for (f, line), s in acc.most_common(top):
    print(f"{100.0 * s / tot:5.1f}%  {f}:{line}: {text_of(f, line)}")
