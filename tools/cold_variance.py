"""Cold config-3 calls back to back vs after an idle pause, with the SM clock sampled around each:
does the cold e2e spread come from the power-capped clock? (GPU box)"""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_0106_b200 as q


def sm_clock():
    out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    return out


n, m = 1 << 24, 256
spec = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
ctx = q.Context(0)
(dv, sp), = ctx.member_streams()
st = torch.cuda.ExternalStream(sp, device=torch.device("cuda", dv))
ctx.price_american(spec, m, n, 42, no_cache=True)
for pause in (0.0, 0.0, 0.0, 2.0, 2.0, 2.0, 0.0, 0.0):
    time.sleep(pause)
    before = sm_clock()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.price_american(spec, m, n, 42, no_cache=True)
    e1.record(st)
    e1.synchronize()
    print("pause %.1f s: cold %.1f ms  (clock/power before: %s, after: %s)" % (pause, e0.elapsed_time(e1), before, sm_clock()))
print("K1 alone: %.1f ms" % min(ctx.time_perm_build(n, 42, m) for _ in range(3)))
