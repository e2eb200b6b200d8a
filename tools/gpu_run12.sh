timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not slow" 2>&1 | tail -3
for tf in 2048 4096; do
 for tma in 1 0; do
   echo "TF=$tf TMA=$tma"
   MOA_FFT_TF=$tf MOA_FFT_TMA=$tma timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
   MOA_FFT_TF=$tf MOA_FFT_TMA=$tma MOA_FFT_FUSE=0 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
 done
done
for sl in "2 1" "4 2" "5 3"; do set -- $sl; MOA_FFT_TF=2048 MOA_FFT_SLOTS=$1 MOA_FFT_LAG=$2 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1; done
MOA_FFT_TF=2048 timeout 120 python tools/perf_probe.py 24 "256,256,256" > gpurun_out/plain12.log 2>&1 && MOA_FFT_TF=2048 ncu --set full --import-source on --clock-control none -k regex:"fused|fft_pass" -s 2 -c 2 -o gpurun_out/prof12 -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu12.log 2>&1
