# re-entry verification: full GPU suite + smoke + default bench line at HEAD
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly --durations=8 > gpurun_out/v1_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/v1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/v1_c4.json 2> gpurun_out/v1_c4.err; echo "c4 rc=$?"
echo done
