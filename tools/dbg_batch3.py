import sys; sys.path.insert(0, ".")
import numpy as np, paper_1205_0106_b200 as q
ctx = q.Context(0)
allspecs = [q.OptionSpec(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, q.OptionKind(0)) for i in range(32) for j in range(32)]
for lg in (16, 17, 18):
    for cnt in (2, 8, 64, 512):
        n = 1 << lg; m = 40
        specs = allspecs[:cnt]
        a = np.array([r.price for r in ctx.price_american_batch(specs, m, n, 42)])
        b = np.array([r.price for r in ctx.price_american_batch(specs, m, n, 42)])
        one = np.array([ctx.price_american(specs[k], m, n, 42).price for k in range(0, cnt, max(1, cnt // 8))])
        print(lg, cnt, "run diffs", np.count_nonzero(a != b), "max rel vs single", np.max(np.abs(a[::max(1, cnt // 8)] - one) / one), flush=True)
