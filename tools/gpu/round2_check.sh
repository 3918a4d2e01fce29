# GPU-box recipe: gpu tests, both bench arms, the sharded path at one rank.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 900 python bench.py --npoints 1000000000 --steps 5 --no-cpu-baseline --no-pageable > gpurun_out/bench_1b_single.json 2> gpurun_out/bench_1b_single.err; tail -3 gpurun_out/bench_1b_single.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --sharded --steps 5 --warmup 3 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err; tail -5 gpurun_out/bench_sharded1.err
cat gpurun_out/bench_1b_single.json gpurun_out/bench_sharded1.json
