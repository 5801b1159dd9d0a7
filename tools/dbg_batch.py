import sys; sys.path.insert(0, ".")
import numpy as np, paper_1205_0106_b200 as q
lg = int(sys.argv[1]); m = int(sys.argv[2]); n = 1 << lg
specs = []
for i in range(32):
    for j in range(32):
        specs.append(q.OptionSpec(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, q.OptionKind((i + j) % 2)))
ctx = q.Context(0)
res = ctx.price_american_batch(specs, m, n, 42, allow_put=True)
bad = []
for k in range(0, 1024, 7):
    one = ctx.price_american(specs[k], m, n, 42, allow_put=True)
    rel = abs(one.price - res[k].price) / max(one.price, 1e-300)
    if rel > 1e-12: bad.append((rel, k, specs[k].strike, specs[k].volatility, int(specs[k].kind), one.price, res[k].price))
bad.sort(reverse=True)
print(len(bad), "bad of", len(range(0,1024,7)))
for b in bad[:10]: print(b)
