import collections, csv, io, os, re, subprocess, sys, tempfile
rep, obj, kre, norm = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
cur_fn, line_of, cur_line, prev_marker = None, {}, None, False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1); continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        if not prev_marker:
            cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        prev_marker = True; continue
    prev_marker = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and cur_fn and re.search(kre, cur_fn):
        line_of[int(m.group(1), 16)] = cur_line
which = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # which captured kernel of the report (0 = first)
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
# a report with several kernels repeats the (kernel line, header) pair per kernel
starts = [k for k, r in enumerate(src) if r and r[0] == "Address"]
h = src[starts[which]]; ix = {k: i for i, k in enumerate(h)}
src = [None] + src[starts[which]:(starts[which + 1] - 1 if which + 1 < len(starts) else len(src))]
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
rows = src[2:]
base = int(rows[0][ix["Address"]], 16)
inst = collections.Counter(); samp = collections.Counter(); ops = collections.defaultdict(collections.Counter)
for r in rows:
    off = int(r[ix["Address"]], 16) - base
    key = line_of.get(off)
    n = int(r[ix["Instructions Executed"]] or 0)
    inst[key] += n
    samp[key] += sum(int(r[ix[s]] or 0) for s in stalls)
    op = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    ops[key][op.split(".")[0]] += n
tot = sum(inst.values())
for key, n in inst.most_common(45):
    print(f"{str(key):28s} {n / norm:7.2f}  samp {samp[key]:7d}  ", dict(ops[key].most_common(5)))
print("total/unit", tot / norm)
