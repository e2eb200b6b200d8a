timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not slow" 2>&1 | tail -3
for tf in 4096 2048; do
 for tma in 1 0; do
  echo "TF=$tf TMA=$tma"
  MOA_FFT_TF=$tf MOA_FFT_TMA=$tma timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
  MOA_FFT_TF=$tf MOA_FFT_TMA=$tma MOA_FFT_FUSE=0 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
 done
done
timeout 120 python tools/perf_probe.py 24 "4096,4096" "2048,8192" 2>&1 | tail -3
export MOA_FFT_FUSE=0
MOA_FFT_TMA=0 MOA_FFT_TF=2048 timeout 120 python tools/perf_probe.py 24 "256,256,256" > gpurun_out/plain9.log 2>&1 && MOA_FFT_TMA=0 MOA_FFT_TF=2048 ncu --set full --import-source on --clock-control none -k regex:fft_pass -s 3 -c 1 -o gpurun_out/prof9_plain -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu9.log 2>&1
