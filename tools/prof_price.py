"""Driver for ncu: warm the tables, then run the pricing step a few times.

usage: python tools/prof_price.py [m] [log2 n] [kind: 0 call, 1 put]"""
import sys
sys.path.insert(0, ".")
import paper_1205_0106_b200 as q
m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kind = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ctx = q.Context(0)
spec = q.OptionSpec(100, 100, 0.05, 0.2, 1.0, kind=q.OptionKind(kind))
ctx.warm(1 << lg, 42, m)
k, st, p, s = ctx.time_device(spec, m, 1 << lg, 42, 3, allow_put=kind == 1)
print("kernel ms", k, "step ms", st, "price", p, s)
