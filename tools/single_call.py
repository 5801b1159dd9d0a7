import time, paper_1205_0106_b200 as q
ctx = q.Context(0)
n, m = 1 << 18, 128
ctx.warm(n, 42, m)
s = q.OptionSpec(100.0, 90.0, 0.05, 0.2, 1.0)
for i in range(4):
    t = time.perf_counter(); r = ctx.price_american(s, m, n, 42); print("call", (time.perf_counter() - t) * 1e3, "ms")
