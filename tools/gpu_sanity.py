"""Quick GPU sanity run: parity of K1/D1/K2 against the oracle at small sizes."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_1205_0106_b200 as q

O = oracle.Oracle()
ctx = q.Context(0)
for n in [1, 2, 3, 8, 17, 1000, 65536, 1 << 20]:
    for seed in [42, 7, 2**63 + 5]:
        g = ctx.permutation(n, seed)[:n]
        r = O.permutation_indices(n, seed)[:n]
        assert (g == r).all(), ("perm", n, seed)
print("perm ok")
for n, seed, dims in [(1000, 42, 5), (1 << 16, 42, 51), (1 << 20, 42, 3)]:
    for d in range(dims) if dims < 10 else [0, 1, 2, 17, 50]:
        gu = ctx.uniforms(n, seed, d)
        ru = O.uniform_dim(d + 1, n, seed, d)
        bad = np.count_nonzero(gu.view(np.uint64) != ru.view(np.uint64))
        assert bad == 0, ("uniform", n, seed, d, bad)
        gz = ctx.normals(n, seed, d)
        rz = np.array([O.moro_inv_cnd(u) for u in ru[:4096]])
        ulps = np.abs(gz[:4096].view(np.int64) - rz.view(np.int64))
        print("normals dim", d, "max ulp", ulps.max())
print("uniforms ok")
spec = q.OptionSpec(100, 100, 0.05, 0.2, 1.0)
for (m, n) in [(1, 1 << 12), (10, 1 << 14), (50, 1 << 16), (100, 1 << 16)]:
    t = time.time()
    rp, rs, rv = O.price_american(100, 100, .05, .2, 1, m, n, 42, want_values=True)
    res = ctx.price_american(spec, m, n, 42)
    gv = ctx.path_values(spec, m, n, 42)
    rel = np.abs(gv - rv) / np.maximum(np.abs(rv), 1e-300)
    print(f"m={m} n={n} gpu {res.price!r} {res.std_error!r} oracle {rp!r} {rs!r} rel {abs(res.price-rp)/rp:.3e} "
          f"path max rel {rel.max():.3e} mismatched {np.count_nonzero(rel > 1e-9)}")
# puts + negative rate + zero vol
for (S, K, r, v, T, kind) in [(100, 100, 0.05, 0.2, 1, 1), (90, 100, -0.02, 0.3, 1, 0), (90, 100, -0.02, 0.3, 1, 1),
                              (100, 100, 0.05, 0.0, 1, 0), (100, 110, 0.0, 0.25, 2, 0)]:
    m, n = 20, 1 << 14
    rp, rs = O.price_american(S, K, r, v, T, m, n, 42, kind=kind, allow_put=True)
    res = ctx.price_american(q.OptionSpec(S, K, r, v, T, q.OptionKind(kind)), m, n, 42, allow_put=True)
    print(f"spec {(S,K,r,v,T,kind)} gpu {res.price!r} oracle {rp!r} rel {abs(res.price-rp)/max(rp,1e-300):.3e} se {res.std_error:.3e} {rs:.3e}")
k, st, p, s = ctx.time_device(spec, 100, 1 << 20, 42, 5)
print("C2 kernel ms", k, "step ms", st, p, s)
t = ctx.time_perm_build(1 << 20, 42, 100)
print("perm build C2 ms", t)
