"""Group ncu_lines output (per-line instruction counts) by enclosing function / region."""
import re, sys
src = open(sys.argv[2]).read().splitlines()
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"^(?:__device__|__global__)[^(]*?\b(\w+)\(", l)
    if m:
        starts.append((i, m.group(1)))
    elif re.match(r"^template <", l) and i < len(src):
        m2 = re.match(r"^(?:__device__|__global__)[^(]*?\b(\w+)\(", src[i])
        if m2:
            starts.append((i + 1, m2.group(1)))
starts.sort()
regions = {}
if len(sys.argv) > 3:
    for spec in sys.argv[3:]:
        name, a, b = spec.split(":")
        regions[name] = (int(a), int(b))


def fn(ln):
    for name, (a, b) in regions.items():
        if a <= ln <= b:
            return name
    name = "?"
    for s, n in starts:
        if s <= ln:
            name = n
    return name


agg = {}
for l in open(sys.argv[1]):
    m = re.match(r"\s*([\d.]+)\s+[\d.]+%\s+samp\s+(\d+)\s+(\S+)", l)
    if not m:
        continue
    v, loc = float(m.group(1)), m.group(3)
    key = fn(int(loc.split(":")[1])) if loc.startswith("kernels.cu:") else loc
    a = agg.setdefault(key, [0.0, 0])
    a[0] += v
    a[1] += int(m.group(2))
tot = sum(a[0] for a in agg.values())
for k, (v, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v:8.2f} {100 * v / tot:5.1f}%  samples {s:8d}  {k}")
