# round-2 evidence pass: Sigma^-1 tolerance probes, then ncu launch lists + full
# captures (tensor-pipe counters) of the c3 and c5 kernels and the c4 pair.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -m gpu -q -s -p no:randomly > gpurun_out/r2_inv.log 2>&1; echo "pytest rc=$?"
grep -E "PARITY|passed|failed|Error" gpurun_out/r2_inv.log | tail -60
C3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
C5="python bench.py --config c5 --lines 16384 --steps 1 --warmup 1"
C4="python bench.py --strips 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
$C3 > gpurun_out/r2_c3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv $C3 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"raww_gram_kernel|raww_scan_kernel|score_tcw_kernel" -c 3 -o gpurun_out/r2_full_c3 -f $C3 > gpurun_out/r2_ncu_c3.log 2>&1
echo "c3 rc=$?"
$C5 > gpurun_out/r2_c5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv $C5 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"gram_raw_kernel|score_tcs_kernel" -c 2 -o gpurun_out/r2_full_c5 -f $C5 > gpurun_out/r2_ncu_c5.log 2>&1
echo "c5 rc=$?"
$C4 > gpurun_out/r2_c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c4.csv $C4 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"gram_raw_kernel|score_tc_kernel|finalize_kernel|topk_mask_pass" -c 4 -o gpurun_out/r2_full_c4 -f $C4 > gpurun_out/r2_ncu_c4.log 2>&1
echo "c4 rc=$?"
ls -la gpurun_out | tail -20
