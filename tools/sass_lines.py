"""Print SASS of a kernel with innermost source line, between two source lines (first occurrence)."""
import re, sys
dis, kre, l0, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
lines = open(dis).read().splitlines()
start = end = None
for i, l in enumerate(lines):
    if re.match(r"\s*\.text\..*" + kre, l):
        start = i
    elif start is not None and re.match(r"\s*\.text\.", l) and i > start + 5:
        end = i
        break
cur, out, prev = None, [], False
for l in lines[start:end]:
    m = re.search(r"line (\d+)", l)
    if "//##" in l and m:
        if not prev:
            cur = int(m.group(1))
        prev = True
        continue
    prev = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        out.append((int(m.group(1), 16), cur, m.group(2).strip()))
first = [i for i, o in enumerate(out) if o[1] == l0][0]
for o in out[first - 5:first + n]:
    print(f"{o[0]:6x} L{o[1]} {o[2]}")
