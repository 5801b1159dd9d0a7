"""Where a cold config-3 call's time goes: wall clock of the C-ABI call vs CUDA events on the
context stream around it, and the K1 build alone. usage (GPU box): python tools/cold_breakdown.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_0106_b200 as q

n, m = 1 << 24, 256
spec = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
ctx = q.Context(0)
(dv, sp), = ctx.member_streams()
st = torch.cuda.ExternalStream(sp, device=torch.device("cuda", dv))
ctx.price_american(spec, m, n, 42, no_cache=True)
for _ in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    ctx.price_american(spec, m, n, 42, no_cache=True)
    e1.record(st)
    e1.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print("cold call: wall %.1f ms, device (stream events) %.1f ms" % (wall, e0.elapsed_time(e1)))
print("K1 + conversion alone: %.1f ms" % min(ctx.time_perm_build(n, 42, m) for _ in range(2)))
k, s_, _, _ = ctx.time_device(spec, m, n, 42, 3)
print("warm pricing: kernel %.2f ms, step %.2f ms" % (k, s_))
