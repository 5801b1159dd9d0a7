"""Config 4: 1024 contracts (32 strikes x 32 vols, calls/puts alternating), 2^18 paths x 128 dates."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1205_0106_b200 as q

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 18
m = int(sys.argv[2]) if len(sys.argv) > 2 else 128
n = 1 << lg
specs = []
for i in range(32):
    for j in range(32):
        specs.append(q.OptionSpec(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, q.OptionKind((i + j) % 2)))
ctx = q.Context(0)
ctx.warm(n, 42, m)
res = ctx.price_american_batch(specs, m, n, 42, allow_put=True)
t0 = time.perf_counter()
reps = 3
for _ in range(reps):
    res = ctx.price_american_batch(specs, m, n, 42, allow_put=True)
dt = (time.perf_counter() - t0) / reps
print(f"batch of {len(specs)}: {dt*1e3:.2f} ms  {len(specs)*n*m/dt:.3e} contract-path-steps/s  launches {ctx.last_launch_count()}")
# check a few against single pricing
worst = 0.0
for k in list(range(0, 1024, 97)) + [1023]:
    one = ctx.price_american(specs[k], m, n, 42, allow_put=True)
    worst = max(worst, abs(one.price - res[k].price) / max(one.price, 1e-300))
print("max rel diff batch vs single", worst)
t0 = time.perf_counter()
for k in range(16):
    ctx.price_american(specs[k], m, n, 42, allow_put=True)
print(f"single fused: {(time.perf_counter()-t0)/16*1e3:.3f} ms per contract")
