"""Per-region instruction counts and warp-stall samples of one kernel from an ncu report.

usage: ncu_regions.py report.ncu-rep kernel.o kernel_regex norm name:first-last[,first-last] ...
Lines are kernels.cu source lines (innermost inlined frame); unmatched lines go to "other".
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, kre, norm = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
regions = []
for spec in sys.argv[5:]:
    name, rngs = spec.split(":")
    for r in rngs.split(","):
        a, b = r.split("-")
        regions.append((name, int(a), int(b)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
cur_fn, line_of, cur_line, prev_marker = None, {}, None, False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        if not prev_marker:
            cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        prev_marker = True
        continue
    prev_marker = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and cur_fn and re.search(kre, cur_fn):
        line_of[int(m.group(1), 16)] = cur_line
src = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
    text=True).stdout)))
h = src[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
rows = src[2:]
base = int(rows[0][ix["Address"]], 16)
inst = collections.Counter()
samp = collections.defaultdict(collections.Counter)


def region(key):
    if key is None:
        return "?"
    f, ln = key
    if f != "kernels.cu":
        return "intrinsics"
    for name, a, b in regions:
        if a <= ln <= b:
            return name
    return "other"


for r in rows:
    off = int(r[ix["Address"]], 16) - base
    reg = region(line_of.get(off))
    inst[reg] += int(r[ix["Instructions Executed"]] or 0)
    for s in stalls:
        samp[reg][s] += int(r[ix[s]] or 0)
tot_s = sum(sum(c.values()) for c in samp.values())
print(f"{'region':12s} {'inst/unit':>9s} {'samples%':>8s}  top stalls (% of all samples)")
for reg, n in sorted(inst.items(), key=lambda x: -sum(samp[x[0]].values())):
    s = samp[reg]
    tops = ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}" for k, v in s.most_common(5) if v)
    print(f"{reg:12s} {n / norm:9.2f} {100 * sum(s.values()) / tot_s:8.1f}  {tops}")
