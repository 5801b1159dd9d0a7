"""Config 3 kernel time and price, FP64 vs the FP32 variant, call and put (GPU box)."""
import sys; sys.path.insert(0, ".")
import paper_1205_0106_b200 as q
ctx = q.Context(0)
n, m = 1 << 24, 256
ctx.warm(n, 42, m)
for kind in (0, 1):
    s = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=q.OptionKind(kind))
    for fp32 in (False, True):
        ctx.time_device(s, m, n, 42, 2, allow_put=kind == 1, fp32=fp32)
        k, st, p, se = ctx.time_device(s, m, n, 42, 5, allow_put=kind == 1, fp32=fp32)
        print("kind", kind, "fp32", fp32, "kernel %.3f ms price %.10f se %.3g" % (k, p, se))
