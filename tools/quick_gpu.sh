#!/bin/bash
# Quick GPU iteration: GPU tests, then bench lines for the 20M configs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for d in uniform_square uniform_disk gaussian circle; do
  timeout 300 python bench.py --steps 10 --warmup 3 --dist $d --no-cpu-baseline > gpurun_out/q_$d.json 2> gpurun_out/q_$d.err
  python -c "
import json; d=json.load(open('gpurun_out/q_$d.json')); r=d['roofline']; pk=r['per_kernel']
print('$d', 'ms', round(d['ms_per_step'],4), 'k1', round(pk['k1_extremes']['ms']*1e3,1), 'k2', round(pk['k2_classify_survivors']['ms']*1e3,1), 'frac', round(r['frac'],3), 'disc', round(r['discard_kernels']['frac'],3))"
done
CHGPU_FINISH_SPLIT_MIN=8 timeout 600 python tests/split_finisher_check.py
for i in 1 2; do timeout 300 python tools/knob_sweep.py X=0 CHGPU_FINISH_SPLIT_MIN=100000000; done
