"""FP32 vs FP64 kernel time and price at config 3 (2^24 x 256) on cuda:0."""
import sys
import paper_1205_0106_b200 as q

ctx = q.Context(0)
n, m = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 24), 256
for kind in (0, 1):
    sp = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=q.OptionKind(kind))
    for fp32 in (False, True):
        k, st, p, se = ctx.time_device(sp, m, n, 42, 5, allow_put=kind == 1, fp32=fp32)
        print(f"kind={kind} fp32={fp32} kernel_ms={k:.3f} step_ms={st:.3f} price={p:.12f} se={se:.3e}", flush=True)
