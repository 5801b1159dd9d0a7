"""FP32-variant prices for a few specs (compare two libraries bit for bit: QMCG_LIB=... python tools/fp32_cmp.py)."""
import sys; sys.path.insert(0, ".")
import paper_1205_0106_b200 as q
ctx = q.Context(0)
out = []
for (s, m, n) in [((100.0, 100.0, 0.05, 0.2, 1.0, 0), 256, 1 << 22), ((90.0, 100.0, 0.03, 0.3, 0.5, 1), 100, 300001),
                  ((100.0, 100.0, -0.02, 0.25, 1.0, 0), 64, 50000), ((100.0, 95.0, 0.05, 0.2, 1.0, 1), 365, 1 << 20)]:
    spec = q.OptionSpec(*s[:5], kind=q.OptionKind(s[5]))
    r = ctx.price_american(spec, m, n, 42, fp32=True, allow_put=True)
    out.append((r.price, r.std_error))
print(out)
