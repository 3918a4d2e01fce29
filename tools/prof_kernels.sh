#!/bin/bash
# usage: tools_prof.sh TAG K1 K2 ...  -- one ncu --set full capture per kernel regex
TAG=$1; shift
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
for K in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/prof_${TAG}_${K} $CMD > gpurun_out/ncu_${TAG}_${K}.log 2>&1
  echo "$K rc=$?"
done
