# Round measurement set (GPU box): bench lines for the four 20M configs (our
# arm + the reference arm), the 1B single-GPU line and the sharded-path line
# at one rank, the launch list of the headline step, ncu --set full captures
# of its kernels with their per-launch DRAM traffic, and a memcheck pass.
# usage: round_measure.sh OUTDIR
O=${1:-gpurun_out/rm}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_uniform_square.json 2> $O/bench_uniform_square.err
for d in uniform_disk gaussian circle; do
  timeout 600 python bench.py --steps 5 --warmup 3 --dist $d --no-cpu-baseline > $O/bench_$d.json 2> $O/bench_$d.err
done
for d in uniform_square uniform_disk gaussian circle; do
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 --dist $d > $O/ref_$d.json 2> $O/ref_$d.err
done
timeout 900 python bench.py --npoints 1000000000 --steps 5 --warmup 3 --no-cpu-baseline --no-pageable > $O/bench_1B_single.json 2> $O/bench_1B_single.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --sharded --steps 5 --warmup 3 > $O/bench_1B_sharded1.json 2> $O/bench_1B_sharded1.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_uniform.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > /dev/null 2>&1
python tools/launch_summary.py $O/launches_uniform.csv > $O/launches_uniform.txt 2>&1
for K in k_extremes_partial k_classify_survivors k_bin_scan k_filter k_spa_small k_spa_finish; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 -o $O/full_$K \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pageable > $O/ncu_$K.log 2>&1
done
# the sort path (20M circle: every point survives and is kept)
for K in k_classify_compact k_upsweep k_colscan k_onesweep k_group_scan k_spa_tile k_convex_check k_convex_emit; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 -o $O/circle_$K \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pageable --dist circle > $O/ncu_circle_$K.log 2>&1
done
python tools/ncu_summary.py $O/circle_*.ncu-rep > $O/ncu_circle_summary.txt 2>&1
python tools/ncu_summary.py $O/full_*.ncu-rep > $O/ncu_full_summary.txt 2>&1
python tools/make_traffic.py $O/traffic.json $O/full_*.ncu-rep > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "
import sys; sys.path.insert(0,'.')
import paper_1508_05488_b200 as P
c=P.Context(0)
for d,n in (('uniform_square',300000),('uniform_disk',100000),('duplicates_heavy',20000),('circle',100000),('gaussian',200000)):
    r=c.convex_hull(P.generate(d,n,1)); print(d, r.stats.n_hull, r.diag.spa_path, r.diag.convex_fast_path)
r=c.convex_hull(P.generate('circle',100000,1)); print('circle again (sort hint)', r.stats.n_hull, r.diag.spa_path)
c.set_spa_path(P.SPA_FILTER_SORTED)
r=c.convex_hull(P.generate('uniform_square',300000,2)); print('filter_sorted', r.stats.n_hull)
c.set_spa_path(P.SPA_SORT)
for cc in (1, 7, 1024):
    r=c.convex_hull(P.generate('uniform_disk',300000,3), P.PipelineConfig(chunk_count=cc)); print('sort path cc', cc, r.stats.n_hull, r.diag.spa_path)
" > $O/memcheck.log 2>&1; echo memcheck=$? >> $O/memcheck.log
# bench lines: the JSON line only (NCCL prints its version first)
for f in $O/*.json; do grep '^{' $f | tail -1 > $f.tmp && mv $f.tmp $f; done
echo done
