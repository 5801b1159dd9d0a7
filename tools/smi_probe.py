"""Does the nvidia-smi clock sampler perturb the timed loop? 50 C-ABI calls, event-timed, with the
sampler off / at 100, 250, 1000 ms (measured: no difference beyond the clock drift under the power cap)."""
import os, subprocess, sys, time
sys.path.insert(0, ".")
import torch
import paper_1205_0106_b200 as q
ctx = q.Context(0)
spec = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
n, m = 1 << 24, 256
ctx.warm(n, 42, m)
(dv, sp), = ctx.member_streams()
st = torch.cuda.ExternalStream(sp, device=torch.device("cuda", dv))
for _ in range(5): ctx.price_american(spec, m, n, 42)
def loop(k=50):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); t0 = time.perf_counter()
    for _ in range(k): ctx.price_american(spec, m, n, 42)
    e1.record(st); e1.synchronize()
    return e0.elapsed_time(e1) / k, (time.perf_counter() - t0) * 1e3 / k
for lms in (None, 100, 250, 1000, None):
    p = None
    if lms:
        p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap", "--format=csv,noheader", "-lms", str(lms)], stdout=subprocess.DEVNULL)
        time.sleep(1.0)
    r = [loop() for _ in range(3)]
    if p: p.terminate(); p.wait()
    print("sampler", lms, ["%.3f/%.3f" % x for x in r])
k, s_, _, _ = ctx.time_device(spec, m, n, 42, 5)
print("kernel %.3f step %.3f" % (k, s_))
