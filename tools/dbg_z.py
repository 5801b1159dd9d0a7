import sys; sys.path.insert(0, ".")
import numpy as np, paper_1205_0106_b200 as q
ctx = q.Context(0)
for lg, m in [(16, 40), (18, 40), (18, 128)]:
    n = 1 << lg
    z1 = ctx.normal_table(n, 42, m); z2 = ctx.normal_table(n, 42, m)
    bad = np.count_nonzero(z1 != z2)
    ref = np.stack([ctx.normals(n, 42, d) for d in range(0, m, 13)])
    err = np.max(np.abs(z1[::13] - ref) / np.maximum(np.abs(ref), 1e-3))
    print(lg, m, "nondeterministic entries", bad, "max rel vs normals()", err)
    if bad:
        idx = np.argwhere(z1 != z2)[:5]; print(idx, z1[tuple(idx[0])], z2[tuple(idx[0])])
