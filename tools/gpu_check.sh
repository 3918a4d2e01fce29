#!/bin/bash
# One GPU session: tests, sanitizer, bench (+cpu baseline), reference arm, launch list.
set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "
import sys; sys.path.insert(0,'.')
import paper_1508_05488_b200 as P
c=P.Context(0)
for d,n in (('uniform_square',300000),('uniform_disk',100000),('duplicates_heavy',20000),('circle',50000)):
    r=c.convex_hull(P.generate(d,n,1)); print(d, r.stats.n_hull)
" > gpurun_out/memcheck.log 2>&1; echo memcheck=$?
tail -3 gpurun_out/memcheck.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
tail -c 600 gpurun_out/bench_ref.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?
