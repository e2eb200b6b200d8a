./tools/l2_probe
MOA_FFT_FUSE=1 timeout 120 python tools/perf_probe.py 24 "256,256,256" > gpurun_out/fplain.log 2>&1 && MOA_FFT_FUSE=1 ncu --set full --import-source on --clock-control none -k regex:"fused|fft_pass" -s 2 -c 2 -o gpurun_out/prof_fused -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu_fused.log 2>&1; tail -3 gpurun_out/ncu_fused.log
