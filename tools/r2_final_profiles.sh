#!/bin/bash
# Round-2 final evidence on one B200 (each profiled command first exits 0 without ncu):
#   the full bench line, the reference arm, the bench launch list (cold-cache, serialised: compare
#   shares), K1 per-launch lists at 2^24 and 2^28, the config-4 batch launch list, and full captures
#   of the headline kernel for the call and the put (config 3).
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_ref_arm.json 2> gpurun_out/r2f_ref_arm.err
echo ref_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline"
$CMD > gpurun_out/r2f_plain.json 2> gpurun_out/r2f_plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_bench_launches.csv $CMD > /dev/null 2>&1
echo launches_rc=$?
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed"
for lg in 24 28; do
  python tools/k1_prof.py $lg > gpurun_out/r2f_k1_$lg.log 2>&1 && \
    ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2f_k1_$lg.csv python tools/k1_prof.py $lg > /dev/null 2>&1
  echo k1_${lg}_rc=$?
done
python tools/c4_batch.py > gpurun_out/r2f_c4.log 2>&1 && \
  ncu --metrics $M,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none \
      -k regex:"walk_group|pairwise|gen_z" -c 9 --csv \
      --log-file gpurun_out/r2f_c4.csv python tools/c4_batch.py > /dev/null 2>&1
echo c4_rc=$?
for kind in 0 1; do
  python tools/prof_price.py 256 24 $kind > gpurun_out/r2f_price_$kind.log 2>&1 && \
    ncu --set full --import-source on --clock-control none -k regex:price_kernel -s 1 -c 1 \
        -o gpurun_out/r2f_price_c3_k$kind python tools/prof_price.py 256 24 $kind > /dev/null 2>&1
  echo price_${kind}_rc=$?
done
lscpu > gpurun_out/r2f_lscpu.txt
