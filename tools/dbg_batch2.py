import sys; sys.path.insert(0, ".")
import numpy as np, paper_1205_0106_b200 as q
lg = int(sys.argv[1]); m = int(sys.argv[2]); n = 1 << lg
specs = [q.OptionSpec(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, q.OptionKind((i + j) % 2)) for i in range(32) for j in range(32)]
ctx = q.Context(0)
a = np.array([r.price for r in ctx.price_american_batch(specs, m, n, 42, allow_put=True)])
b = np.array([r.price for r in ctx.price_american_batch(specs, m, n, 42, allow_put=True)])
one = np.array([ctx.price_american(specs[k], m, n, 42, allow_put=True).price for k in range(0, 1024, 7)])
print("run-to-run diffs", np.count_nonzero(a != b), "max rel vs single", np.max(np.abs(a[::7] - one) / one))
