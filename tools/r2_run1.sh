set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_c4.json; tail -5 gpurun_out/r2_bench_c4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r2_bench_c5_nccl.json 2> gpurun_out/r2_bench_c5_nccl.err; echo "c5 rc=$?"
tail -c 1500 gpurun_out/r2_bench_c5_nccl.json; tail -5 gpurun_out/r2_bench_c5_nccl.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/r2_bench_ref.json
