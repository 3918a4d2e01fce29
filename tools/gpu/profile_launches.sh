# Launch list (per-kernel durations, serialised, cold caches) of the bench
# step, plus the per-call timeline.
set -x
mkdir -p gpurun_out
python tools/gpu/timeline.py > gpurun_out/timeline.json 2>&1; cat gpurun_out/timeline.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
