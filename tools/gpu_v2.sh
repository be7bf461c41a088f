# closing check: full GPU suite + smoke + the default bench line + c5/c1/c2 lines
cd "$(dirname "$0")/.."
bash tools/gpu_v1.sh
for c in c5 c1 c2; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"; done
