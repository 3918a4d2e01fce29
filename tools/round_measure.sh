#!/bin/bash
# Round measurement: bench lines for the four 20M configs (ours + reference
# arm), launch list, full ncu captures of the top kernels (uniform), their
# per-launch DRAM traffic, and a memcheck pass.
O=gpurun_out/rm
mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_uniform_square.json 2> $O/bench_uniform_square.err
for d in uniform_disk gaussian circle; do
  timeout 600 python bench.py --steps 5 --warmup 3 --dist $d --no-cpu-baseline > $O/bench_$d.json 2> $O/bench_$d.err
done
for d in uniform_square uniform_disk gaussian circle; do
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --dist $d > $O/ref_$d.json 2> $O/ref_$d.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_uniform.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/launches_uniform.csv > $O/launches_uniform.txt 2>&1
for K in k_classify_survivors k_filter k_extremes_partial k_bin_scan k_spa_chunks k_spa_emit k_bin_sort_warp; do
  ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 -o $O/full_$K \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$K.log 2>&1
done
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/ncu_full_summary.txt 2>&1
python tools/make_traffic.py $O/traffic.json $O/full_*.ncu-rep > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "
import sys; sys.path.insert(0,'.')
import paper_1508_05488_b200 as P
c=P.Context(0)
for d,n in (('uniform_square',300000),('uniform_disk',100000),('duplicates_heavy',20000),('circle',100000),('gaussian',200000)):
    r=c.convex_hull(P.generate(d,n,1)); print(d, r.stats.n_hull, r.diag.spa_path, r.diag.convex_fast_path)
" > $O/memcheck.log 2>&1; echo memcheck=$? >> $O/memcheck.log
echo done
