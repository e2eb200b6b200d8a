timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
P="timeout 120 python tools/perf_probe.py"
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo fuse2; MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
echo plain-26; $P 26 "" 2>&1 | tail -1
timeout 300 python bench.py --steps 10 > gpurun_out/bench_f.log 2>&1; tail -c 1500 gpurun_out/bench_f.log
MOA_FFT_FUSE=2 $P 24 "256,256,256" > gpurun_out/f2plain.log 2>&1 && MOA_FFT_FUSE=2 ncu --set full --import-source on --clock-control none -k regex:"fused|fft_pass" -s 3 -c 2 -o gpurun_out/prof_f2c -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu_f2.log 2>&1; tail -2 gpurun_out/ncu_f2.log
