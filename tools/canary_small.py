"""Small invocations of every kernel family (K1 table builds incl. the binned scatter, K2 pricing:
call / put / FP32 / r < 0 / sigma = 0 / streamed windows, K3 trees, K4 batch walk, the European
kernel, the exports, a device group), each followed by the guard-region check of every device
buffer (run with QMCG_CANARY=1): tests/test_gpu_bounds.py."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1205_0106_b200 as q  # noqa: E402

ctx = q.Context(0)
check = q.qmcg.check_canaries
spec = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
put = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, q.OptionKind.Put)
out = []
out.append(ctx.price_american(spec, 20, 3001, 42).price)                       # K1 + K2 + K3
check()
out.append(ctx.price_american(put, 20, 3001, 42, allow_put=True).price)        # put walk
check()
out.append(ctx.price_american(spec, 20, 3001, 42, fp32=True).price)            # FP32 kernel
check()
out.append(ctx.price_american(q.OptionSpec(100.0, 95.0, -0.02, 0.3, 1.0), 12, 2049, 7).price)  # r < 0
check()
out.append(ctx.price_american(q.OptionSpec(100.0, 100.0, 0.05, 0.0, 1.0), 6, 100, 7).price)   # sigma = 0
check()
ctx.set_table_budget(8 * 8 * 4224)                                              # streamed date windows
out.append(ctx.price_american(spec, 40, 4097, 42).price)
check()
ctx.set_table_budget(0)
specs = [q.OptionSpec(100.0, 80 + 5 * i, 0.05, 0.1 + 0.05 * j, 1.0, q.OptionKind((i + j) % 2))
         for i in range(6) for j in range(4)]
out.append(ctx.price_american_batch(specs, 16, 4096, 42, allow_put=True)[0].price)  # K4 gen_z + walk + leaves
check()
out.append(ctx.mc_european_price(spec, 5000, 42).price)
check()
ctx.uniform_rows(2000, 42, 3, 5)
check()
ctx.normal_table(2000, 42, 9)
check()
ctx.permutation(70001, 12345)
check()
ctx.permutation((1 << 25) + 3, 777)  # K1's binned scatter (n >= 2^25)
check()
ctx.simulate_batch(spec, 5, 1000, 42)
check()
ctx.sweep_batch(spec, 5, 1000, 42)
check()
g = q.Context(devices=[0, 0])                                                   # group: sharded build + peer copies
out.append(g.price_american(spec, 24, 5000, 42).price)
check()
g.close()
ctx.close()
check()
print("canary_small ok", np.array(out))
