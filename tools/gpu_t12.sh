# session-3 evidence pass: full GPU suite, benches (c4 default, c3, c5, c2, c1), launch lists,
# ncu --set full of the kernels changed this session
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/t12_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t12_pytest.log
timeout 900 python bench.py > gpurun_out/t12_c4.json 2> gpurun_out/t12_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c3 > gpurun_out/t12_c3.json 2> gpurun_out/t12_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c5 --no-cpu > gpurun_out/t12_c5.json 2> gpurun_out/t12_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/t12_c2.json 2> gpurun_out/t12_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/t12_c1.json 2> gpurun_out/t12_c1.err; echo "c1 rc=$?"
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
C4="python bench.py --strips 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t12_launches_c3.csv $C3 > /dev/null 2>&1; echo "ncu c3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t12_launches_c4.csv $C4 > /dev/null 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fw_factor|fw_trinv|raww_gram|score_tcw" -c 4 -o gpurun_out/t12_full_c3 -f $C3 > /dev/null 2>&1; echo "ncu full c3 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"calibrate_bin_tiled" -c 1 -o gpurun_out/t12_full_calbin -f python tools/time_calbin.py > /dev/null 2>&1; echo "ncu calbin rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gram_tc_kernel" -c 1 -o gpurun_out/t12_full_gtc -f python tools/cliff_case.py --gains > /dev/null 2>&1; echo "ncu gtc rc=$?"
timeout 600 python tools/time_cliff.py > gpurun_out/t12_cliff.txt 2>&1
PYTHONPATH=. timeout 600 python tools/stage_probe.py > gpurun_out/t12_stage.txt 2>&1
ls gpurun_out | head -50
