# One ncu --set full capture per kernel regex of the 20M uniform bench step.
# usage: ncu_full.sh TAG KERNEL...
TAG=$1; shift
mkdir -p gpurun_out
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 \
    -o "gpurun_out/full_${TAG}_${K//[^A-Za-z0-9_]/_}" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pageable ${BENCH_ARGS:-} \
    > "gpurun_out/ncu_${TAG}_${K//[^A-Za-z0-9_]/_}.log" 2>&1
  echo "$K rc=$?"
done
python tools/ncu_summary.py gpurun_out/full_${TAG}_*.ncu-rep > gpurun_out/ncu_${TAG}_summary.txt 2>&1
cat gpurun_out/ncu_${TAG}_summary.txt
