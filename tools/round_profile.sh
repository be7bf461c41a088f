#!/bin/bash
# Round-end measurement pass on one B200 (run under gpurun): bench lines of every
# config, the c4 launch list and one ncu --set full capture of the two c4 passes.
# Outputs land in gpurun_out/; copy the summaries into profiles/.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c5 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4.csv \
  python bench.py --strips 2 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"score_tc_kernel|gram_raw_kernel" \
  -c 2 -o gpurun_out/full_c4 -f python tools/time_score.py > gpurun_out/ncu_full.log 2>&1
