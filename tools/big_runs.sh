#!/bin/bash
# Shard-size and full-size runs: 125M (the per-GPU shard of the 1B config)
# and 1B uniform on one GPU (bench lines), plus 1B and 200M disk parity
# against the reference.
mkdir -p gpurun_out/big
timeout 900 python bench.py --n 125000000 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/big/bench_125M.json 2> gpurun_out/big/bench_125M.err; echo b125=$?
timeout 1200 python bench.py --n 1000000000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/big/bench_1B.json 2> gpurun_out/big/bench_1B.err; echo b1B=$?
timeout 1500 python tests/big_parity.py 1e9 > gpurun_out/big/parity_1B.json 2> gpurun_out/big/parity_1B.err; echo p1B=$?
timeout 900 python tests/big_parity.py 2e8 uniform_disk 7 > gpurun_out/big/parity_200M_disk.json 2> gpurun_out/big/parity_200M_disk.err; echo p200d=$?
free -g | head -2
