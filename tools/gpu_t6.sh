cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/time_cliff.py 2>&1 | tail -5
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/t6_c1.log 2>&1; tail -1 gpurun_out/t6_c1.log | cut -c1-300
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/t6_c2.log 2>&1; tail -1 gpurun_out/t6_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in d if k not in ('parity','config')})"
