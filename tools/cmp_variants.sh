# usage (on the GPU box): bash tools/cmp_variants.sh [variant ...]  -- time + ncu counts of the C3 call kernel
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in default "$@"; do
  if [ "$v" = default ]; then L=""; else L="QMCG_LIB=paper_1205_0106_b200/_variants/libqmcg_$v.so"; fi
  echo "== $v"
  env $L python tools/prof_price.py 256 24
  env $L ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:price_kernel -s 1 -c 1 python tools/prof_price.py 256 24 2>&1 | grep -E "inst_executed|duration|fp64|issue"
done
