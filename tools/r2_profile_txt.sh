#!/bin/bash
# Turn the gpurun_out/r2f_* outputs of tools/r2_final_profiles.sh into the committed profiles/ summaries.
set -e
cd "$(dirname "$0")/.."
G=gpurun_out
{
echo "# ncu --metrics gpu__time_duration.sum --clock-control none: every launch of"
echo "#   python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline   (final round-2 build, one B200; tools/r2_final_profiles.sh)"
echo "# cold-cache and serialised (compare SHARES, not absolutes). K1 launches (draws .. chase; uniforms_kernel = the"
echo "# uniform-table conversion): time_perm_build + the cold e2e calls (5 x 256 tables + extras); price_kernel<0>: warm-up,"
echo "# timed steps, time_device and the cold calls. dfma_probe_kernel = bench.py's live FP64 issue-peak probe (roofline)."
python tools/launch_table.py agg $G/r2f_bench_launches.csv
} > profiles/r2_bench_launches.txt
{
echo "# ncu launch list of tools/k1_prof.py 24 and 28 (two tables each, built twice: untimed + timed; serialised under ncu)."
echo "# Final round-2 K1: draws -> CUB sort of j's high bits (16-bit keys, 2 onesweep passes at 2^24; 32-bit keys, 3 passes at"
echo "# 2^28) -> span starts -> span sweep -> chase (-> bin + scatter from 2^25) -> uniforms_kernel (the f64 uniform-table"
echo "# conversion; dims 0 and 1 = the longest digit expansions, 24 and 16 digits; ~84 us averaged over config 3's 256 dims)."
echo "## n = 2^24"
python tools/launch_table.py agg $G/r2f_k1_24.csv
echo "## n = 2^28"
python tools/launch_table.py agg $G/r2f_k1_28.csv
echo "## per launch, n = 2^24 (first table)"
python tools/launch_table.py each $G/r2f_k1_24.csv | head -11
} > profiles/r2_k1_launches.txt
{
echo "# ncu launch list of one config-4 batch call (tools/c4_batch.py: 1024 contracts = 32 strikes x 32 vols, calls/puts"
echo "# alternating, 2^18 paths x 128 dates; uniform tables warm), final round-2 build: prefix sums (gen_z<1>), the grouped"
echo "# walks (calls, puts) and the pairwise trees of the 1024 per-contract value rows"
python tools/launch_table.py each $G/r2f_c4.csv
} > profiles/r2_c4_launches.txt
for k in 0 1; do
  python tools/ncu_summary.py $G/r2f_price_c3_k$k.ncu-rep 134217728 > /tmp/r2sum_$k.txt 2>&1
  python tools/ncu_lines_top.py $G/r2f_price_c3_k$k.ncu-rep paper_1205_0106_b200/libqmcg.so "price_kernelILi${k}ELb0ELb0ELb0E" 134217728 > /tmp/r2lines_$k.txt 2>&1
done
{
echo "# ncu --set full --import-source on --clock-control none, $G/r2f_price_c3_k0.ncu-rep: price_kernel<0> (call),"
echo "# config 3 (2^24 paths x 256 dates, uniform table warm), final round-2 build (tools/r2_final_profiles.sh);"
echo "# per-unit counts are per warp-date (2^32 / 32). Round 1 (permutation tables, digits in K2,"
echo "# profiles/r1_c3_price_kernel_ncu.txt): 104.5 warp-inst per warp-date, 31.2 FP64 per path-step, 16.53 ms, barrier stalls 16.4%."
cat /tmp/r2sum_0.txt
echo
echo "# per source line (kernels.cu of this commit; asm statements attribute to their last line), warp instructions per warp-date, stall samples, top opcodes"
cat /tmp/r2lines_0.txt
} > profiles/r2_c3_price_kernel_ncu.txt
{
echo "# ncu --set full --import-source on --clock-control none, $G/r2f_price_c3_k1.ncu-rep: price_kernel<1> (put),"
echo "# config 3 (2^24 paths x 256 dates, uniform table warm), final round-2 build; per-unit counts per warp-date (2^32 / 32)."
echo "# The put's walk step (walk_date<1>: the record-dominance bound of record_dominates<1>, margin folded into u1) costs"
echo "# ~18 warp-inst per warp-date against the call's 7.5; generation is identical. Round 1: profiles/r1_put_c3_price_kernel_ncu.txt."
cat /tmp/r2sum_1.txt
echo
echo "# per source line (kernels.cu of this commit), warp instructions per warp-date, stall samples, top opcodes"
cat /tmp/r2lines_1.txt
} > profiles/r2_put_c3_price_kernel_ncu.txt
cp $G/r2f_bench.json profiles/r2_bench_1gpu.json
cp $G/r2f_ref_arm.json profiles/r2_reference_arm.json
cp $G/r2f_lscpu.txt profiles/r2_lscpu.txt
cp profiles/roofline_inputs.json /tmp/ri_old.json
python tools/roofline_inputs.py $G/r2f_price_c3_k0.ncu-rep 16777216 256 profiles/roofline_inputs.json /tmp/ri.txt > /dev/null
python - <<'PY'
import json
old = json.load(open('/tmp/ri_old.json')); new = json.load(open('profiles/roofline_inputs.json'))
new['note'] = old['note']
json.dump(new, open('profiles/roofline_inputs.json', 'w'), indent=1)
PY
echo done
