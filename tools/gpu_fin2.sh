# short evidence refresh after a gram_raw change: c1/c2/c5 bench lines, c4 launch list and
# ncu full capture of the two c4 passes, cliff timings (the c4 line + suite come from gpu_v1.sh)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c5 c2 c1; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"; done
C4="python bench.py --strips 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
$C4 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c4.csv $C4 > /dev/null 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_raw_kernel|score_tc_kernel|topk_mask_pass" -c 3 -o gpurun_out/fin_full_c4 -f $C4 > /dev/null 2>&1; echo "ncu full c4 rc=$?"
timeout 600 python tools/time_cliff.py > gpurun_out/fin_cliff.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
echo done
