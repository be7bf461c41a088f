# session-4 check on a fresh container: GPU suite + smoke + c4 bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/s4_c4.json 2> gpurun_out/s4_c4.err; echo "c4 rc=$?"; cat gpurun_out/s4_c4.json | head -c 600
PYTHONPATH=. timeout 300 python tools/time_finalize.py > gpurun_out/s4_fin.txt 2>&1; tail -5 gpurun_out/s4_fin.txt
echo done
