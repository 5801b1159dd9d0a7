#!/bin/bash
# A/B of the leaf-sum kernel (K3 leaves) at config 4: per-launch ncu durations per library variant.
for L in paper_1205_0106_b200/_variants/libqmcg_base.so paper_1205_0106_b200/_variants/libqmcg_leaf2lane.so; do
  n=$(basename $L .so)
  QMCG_LIB=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pairwise_leaves --csv \
    --log-file gpurun_out/leaf_$n.csv python tools/c4_batch.py > gpurun_out/leaf_$n.log 2>&1
  QMCG_LIB=$L python tools/c4_batch.py > gpurun_out/leafplain_$n.log 2>&1
done
