"""Attribute ncu per-instruction execution counts to CUDA source lines.

usage: ncu_lines.py report.ncu-rep kernel.o kernel_regex [norm]
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, kre = sys.argv[1], sys.argv[2], sys.argv[3]
norm = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
# map (function, offset) -> innermost source line (file:line)
cur_fn, line_of = None, {}
cur_line = None
prev_was_marker = False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        if not prev_was_marker:  # first marker of a group = innermost source line
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        prev_was_marker = True
        continue
    prev_was_marker = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and cur_fn and re.search(kre, cur_fn):
        line_of[int(m.group(1), 16)] = cur_line
src = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
h = src[1]
ix = {k: i for i, k in enumerate(h)}
rows = src[2:]
# a report with several kernels repeats the header: keep the first kernel's rows
for k, r in enumerate(rows):
    if r and r[0] == "Kernel Name":
        rows = rows[:k]
        break
base = int(rows[0][ix["Address"]], 16)
agg = collections.Counter()
samp = collections.Counter()
for r in rows:
    off = int(r[ix["Address"]], 16) - base
    ex = int(r[ix["Instructions Executed"]] or 0)
    key = line_of.get(off, "?")
    agg[key] += ex
    samp[key] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(agg.values())
print("total", tot / norm)
srcfile = None
for k, c in agg.most_common(int(os.environ.get("TOPN", "45"))):
    text = ""
    if k != "?":
        f, l = k.split(":")
        p = os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "csrc", f)
        if os.path.exists(p):
            text = open(p).read().splitlines()[int(l) - 1].strip()[:90]
    print(f"{c / norm:9.2f} {100 * c / tot:5.1f}% samp {samp[k]:6d} {k:18s} {text}")
