# usage (GPU box): bash tools/c4_variants.sh [variant ...] -- config-4 batch time per library variant
for v in default "$@"; do
  if [ "$v" = default ]; then L=""; else L="QMCG_LIB=paper_1205_0106_b200/_variants/libqmcg_$v.so"; fi
  env $L PYTHONPATH=. python tools/c4_batch.py > gpurun_out/c4_$v.txt 2>&1
  echo "== $v: $(head -2 gpurun_out/c4_$v.txt | tr '\n' ' ')"
done
