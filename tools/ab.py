"""A/B timing of kernel variants: round-robin over libraries, one fresh process per
(variant, round), each reporting the per-rep kernel times; prints min and median per variant.

usage (GPU box): python tools/ab.py [rounds] [m] [log2 n] [kind]   (variants: default + _variants/*.so)
"""
import glob, os, statistics, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = sys.argv[2] if len(sys.argv) > 2 else "256"
lg = sys.argv[3] if len(sys.argv) > 3 else "24"
kind = sys.argv[4] if len(sys.argv) > 4 else "0"
libs = [""] + sorted(glob.glob(os.path.join(root, "paper_1205_0106_b200", "_variants", "*.so")))
child = r'''
import sys; sys.path.insert(0, "%s")
import paper_1205_0106_b200 as q
ctx = q.Context(0)
kind = int(sys.argv[3])
s = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=q.OptionKind(kind))
n = 1 << int(sys.argv[2]); m = int(sys.argv[1])
ctx.warm(n, 42, m)
ctx.time_device(s, m, n, 42, 2, allow_put=kind == 1)
for _ in range(6):
    k, st, p, se = ctx.time_device(s, m, n, 42, 1, allow_put=kind == 1)
    print(k, p)
''' % root
res = {l: [] for l in libs}
for r in range(rounds):
    for l in libs:
        env = dict(os.environ)
        if l:
            env["QMCG_LIB"] = l
        out = subprocess.run([sys.executable, "-c", child, m, lg, kind], env=env, capture_output=True, text=True)
        for line in out.stdout.split("\n"):
            if line.strip():
                k, p = line.split()
                res[l].append(float(k))
        if out.returncode:
            print(os.path.basename(l) or "default", out.stderr[-400:])
for l in libs:
    v = res[l]
    if v:
        print(f"{os.path.basename(l) or 'default':28s} min {min(v):8.3f}  med {statistics.median(v):8.3f}  n {len(v)}")
