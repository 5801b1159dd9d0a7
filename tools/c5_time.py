"""Config 5 wall time on one GPU: 2^28 x 365 FP32 (streamed tables), and the K1 share."""
import time
import paper_1205_0106_b200 as q

ctx = q.Context(0)
sp = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
n, m = 1 << 28, 365
ctx.price_american(sp, 16, 1 << 12, 42)  # load the module
t = time.perf_counter()
r = ctx.price_american(sp, m, n, 42, fp32=True)
wall = time.perf_counter() - t
print(f"C5 fp32: price={r.price:.10f} se={r.std_error:.3e} wall={wall:.3f}s windows={ctx.last_window_count()} "
      f"path-steps/s={n * m / wall:.3e}", flush=True)
ctx.clear_cache()
for dims in (4, 16):
    ms = ctx.time_perm_build(n, 42, dims)
    print(f"K1 2^28 x {dims}: {ms:.1f} ms ({ms / dims:.2f} ms/table)", flush=True)
    ctx.clear_cache()
