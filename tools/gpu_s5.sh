mkdir -p gpurun_out
for r in 1 2; do python tools/time_sc_libs.py tools/_var/sc_lane0.so tools/_var/sc_elect.so; done > gpurun_out/s5_sc.log 2>&1; cat gpurun_out/s5_sc.log
for r in 1 2; do python tools/time_gr_libs.py tools/_var/gr_lane0.so tools/_var/gr_elect.so; done > gpurun_out/s5_gr.log 2>&1; cat gpurun_out/s5_gr.log
bash tools/fp_profile.sh > gpurun_out/s5_fp.log 2>&1; cat gpurun_out/s5_fp.log | tail -5
