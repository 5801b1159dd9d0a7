#!/bin/bash
# Round-2 evidence on one B200: the bench launch list (cold-cache, serialised: compare shares), a
# full capture of the headline kernel (price_kernel, call, config 3), K1 per-launch list at 2^24,
# config-4 batch launch list. Every profiled command first exits 0 without ncu.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline"
$CMD > gpurun_out/r2_plain.json 2> gpurun_out/r2_plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv $CMD > gpurun_out/r2_ncu_launches.log 2>&1
echo launches_rc=$?
python tools/prof_price.py 256 24 > gpurun_out/r2_price_plain.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:price_kernel -s 1 -c 1 -o gpurun_out/r2_price_c3 python tools/prof_price.py 256 24 > gpurun_out/r2_price_ncu.log 2>&1
echo price_rc=$?
python tools/k1_prof.py 24 > gpurun_out/r2_k1_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2_k1_launches.csv python tools/k1_prof.py 24 > /dev/null 2>&1
echo k1_rc=$?
python tools/c4_batch.py > gpurun_out/r2_c4_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 12 --csv --log-file gpurun_out/r2_c4_launches.csv python tools/c4_batch.py > /dev/null 2>&1
echo c4_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_arm.json 2> gpurun_out/r2_ref_arm.err
echo ref_rc=$?
lscpu > gpurun_out/r2_lscpu.txt
