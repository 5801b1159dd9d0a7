#!/bin/bash
# ncu evidence beyond the headline kernel: K1 (cold table build, 2^24), config 4 batch kernels,
# and the put variant of price_kernel at config 3. Each program first runs without ncu.
set -x
mkdir -p gpurun_out
python tools/k1_prof.py 24 > gpurun_out/x_k1.log 2>&1 && \
  ncu --set full --clock-control none -k regex:fy_ -c 12 -o gpurun_out/prof_k1_24 python tools/k1_prof.py 24 > gpurun_out/x_k1_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1_launches.csv python tools/k1_prof.py 24 > /dev/null 2>&1
timeout 300 python tools/c4_batch.py > gpurun_out/x_c4.log 2>&1 && \
  ncu --set full --clock-control none -k regex:"walk_group|gen_z" -c 4 -o gpurun_out/prof_c4 python tools/c4_batch.py > gpurun_out/x_c4_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/c4_batch.py > /dev/null 2>&1
cat > /tmp/put.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_1205_0106_b200 as q
ctx = q.Context(0); s = q.OptionSpec(100, 100, 0.05, 0.2, 1.0, kind=q.OptionKind.Put)
ctx.warm(1 << 24, 42, 256)
print(ctx.time_device(s, 256, 1 << 24, 42, 2, allow_put=True))
PY
python /tmp/put.py > gpurun_out/x_put.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:price_kernel -s 1 -c 1 -o gpurun_out/prof_put_c3 python /tmp/put.py > gpurun_out/x_put_ncu.log 2>&1
ls -la gpurun_out
