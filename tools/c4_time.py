"""Config-4 batch device time (CUDA events on the context's stream), min / median of 10 batches.
usage (GPU box): [QMCG_LIB=...] python tools/c4_time.py"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_0106_b200 as q

n, m = 1 << 18, 128
specs = [q.OptionSpec(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, q.OptionKind((i + j) % 2))
         for i in range(32) for j in range(32)]
ctx = q.Context(0)
ctx.warm(n, 42, m)
(dv, sp), = ctx.member_streams()
st = torch.cuda.ExternalStream(sp, device=torch.device("cuda", dv))
for _ in range(2):
    ctx.price_american_batch(specs, m, n, 42, allow_put=True)
t = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.price_american_batch(specs, m, n, 42, allow_put=True)
    e1.record(st)
    e1.synchronize()
    t.append(e0.elapsed_time(e1))
print(os.path.basename(os.environ.get("QMCG_LIB", "")) or "default", "min %.3f med %.3f ms" % (min(t), statistics.median(t)))
