"""Kernel time of the config-3 call and put (tables warm)."""
import paper_1205_0106_b200 as q
ctx = q.Context(0)
n = 1 << 24
for kind in (0, 1):
    s = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=q.OptionKind(kind))
    k, st, p, se = ctx.time_device(s, 256, n, 42, 5, allow_put=kind == 1)
    print(f"kind={kind} kernel_ms={k:.3f} price={p:.15f} se={se:.6e}")
