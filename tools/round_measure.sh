#!/bin/bash
# Round measurement: bench lines for the four 20M configs (ours + reference
# arm), launch list and full ncu captures of the top kernels (uniform).
mkdir -p gpurun_out/rm
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/rm/bench_uniform.json 2> gpurun_out/rm/bench_uniform.err
for d in uniform_disk gaussian circle; do
  timeout 600 python bench.py --steps 5 --warmup 3 --dist $d --no-cpu-baseline > gpurun_out/rm/bench_$d.json 2> gpurun_out/rm/bench_$d.err
done
for d in uniform_square uniform_disk gaussian circle; do
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --dist $d > gpurun_out/rm/ref_$d.json 2> gpurun_out/rm/ref_$d.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/rm/launches_uniform.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/rm/launches_uniform.csv > gpurun_out/rm/launches_uniform.txt 2>&1
for K in k_classify_compact k_filter k_extremes_partial; do
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/rm/full_$K \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/rm/ncu_$K.log 2>&1
done
python tools/ncu_summary.py gpurun_out/rm/full_*.ncu-rep > gpurun_out/rm/ncu_full_summary.txt 2>&1
for K in k_classify_compact k_filter k_extremes_partial; do
  ncu -i gpurun_out/rm/full_$K.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/rm/raw_$K.csv 2>&1
done
echo done
