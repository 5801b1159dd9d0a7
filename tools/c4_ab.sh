#!/bin/bash
# config-4 batch: fused leaves (default) vs the leaves kernel, alternating fresh processes
for r in 1 2 3; do
  echo "fused:   $(python tools/c4_batch.py | head -1)"
  echo "unfused: $(QMCG_NO_FUSED_LEAVES=1 python tools/c4_batch.py | head -1)"
done
