#!/bin/bash
# usage: tools_prof.sh TAG  -- captures one launch of each hot kernel with ncu --set full
TAG=${1:-r}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
for K in k_classify_compact k_onesweep k_group_scan k_spa k_extremes_partial k_extremes_final k_hist; do
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/prof_${TAG}_${K} $CMD > gpurun_out/ncu_${TAG}_${K}.log 2>&1
  echo "$K rc=$?"
done
