"""ncu driver for the config-3 pricing kernel: warm tables, then price (call) a few times."""
import sys
sys.path.insert(0, ".")
import paper_1205_0106_b200 as q
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
m = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctx = q.Context(0)
s = q.OptionSpec(100, 100, 0.05, 0.2, 1.0)
ctx.warm(1 << lg, 42, m)
for _ in range(3):
    r = ctx.price_american(s, m, 1 << lg, 42)
print(r.price, r.std_error)
