# end-of-round evidence pass: full GPU suite + smoke, every bench line (c4 default incl. CPU
# baseline and e2e, the reference arm, c1/c2/c3/c5), launch lists and ncu captures
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
for c in c3 c5 c2 c1; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"; done
C4="python bench.py --strips 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
C5="python bench.py --config c5 --lines 16384 --steps 1 --warmup 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c4.csv $C4 > /dev/null 2>&1; echo "ncu c4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c3.csv $C3 > /dev/null 2>&1; echo "ncu c3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c5.csv $C5 > /dev/null 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_raw_kernel|score_tc_kernel|topk_mask_pass" -c 3 -o gpurun_out/fin_full_c4 -f $C4 > /dev/null 2>&1; echo "ncu full c4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_raw_kernel|score_tcs_kernel" -c 2 -o gpurun_out/fin_full_c5 -f $C5 > /dev/null 2>&1; echo "ncu full c5 rc=$?"
timeout 600 python tools/time_cliff.py > gpurun_out/fin_cliff.txt 2>&1
PYTHONPATH=. timeout 600 python tools/stage_probe.py > gpurun_out/fin_stage.txt 2>&1
echo done
