timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variant" 2>&1 | tail -3
P="timeout 120 python tools/perf_probe.py"
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo fuse2; MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
echo fuse3; MOA_FFT_FUSE=3 $P 24 "256,256,256" 2>&1 | tail -1
echo fuse2-lag1; MOA_FFT_FUSE=2 MOA_FFT_SLOTS=3 MOA_FFT_LAG=1 $P 24 "256,256,256" 2>&1 | tail -1
echo tma; MOA_FFT_TMA=1 $P 24 "256,256,256" 2>&1 | tail -1
echo tma-fuse1; MOA_FFT_TMA=1 MOA_FFT_FUSE=1 $P 24 "256,256,256" 2>&1 | tail -1
echo plain-128; $P 24 "128,256,512" 2>&1 | tail -1
echo plain-26; $P 26 "1024,256,256" "64,16,256,256" "16,64,256,256" 2>&1 | tail -3
MOA_FFT_FUSE=2 $P 24 "256,256,256" > gpurun_out/f2plain.log 2>&1 && MOA_FFT_FUSE=2 ncu --set full --import-source on --clock-control none -k regex:"fused" -s 1 -c 1 -o gpurun_out/prof_f2b -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu_f2.log 2>&1; tail -2 gpurun_out/ncu_f2.log
