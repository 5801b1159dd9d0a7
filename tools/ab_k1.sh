#!/bin/bash
# usage (GPU box): bash tools/ab_k1.sh [log2 n] -- K1 time per table for the default library and every _variants/*.so
lg=${1:-24}
export PYTHONPATH=$PWD
for l in "" paper_1205_0106_b200/_variants/*.so; do
  for r in 1 2 3; do
    QMCG_LIB=$l python -c "
import paper_1205_0106_b200 as q
ctx = q.Context(0)
ctx.time_perm_build(1 << $lg, 42, 2)
print('${l:-default}', [round(ctx.time_perm_build(1 << $lg, 42, 8) / 8, 3) for _ in range(2)])"
  done
done
