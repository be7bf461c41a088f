# session-3 first pass: full GPU suite, default bench (c4), c3 and c5 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t1_pytest.log
timeout 900 python bench.py > gpurun_out/t1_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/t1_c4.log
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/t1_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/t1_c3.log
timeout 600 python bench.py --config c5 --no-cpu > gpurun_out/t1_c5.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/t1_c5.log
