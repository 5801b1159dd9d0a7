"""Kernel time vs number of dates at 2^24 paths: the marginal cost of each 8-date tile."""
import paper_1205_0106_b200 as q
ctx = q.Context(0)
s = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
n = 1 << 24
ctx.warm(n, 42, 256)
prev = 0.0
for m in (8, 16, 24, 32, 40, 64, 128, 256):
    k, st, p, se = ctx.time_device(s, m, n, 42, 3)
    print(f"m={m:4d} kernel_ms={k:8.3f}  per-8-date since previous: {8 * (k - prev) / (m - (m - 8 if m <= 40 else {64: 40, 128: 64, 256: 128}[m])):.3f}")
    prev = k
