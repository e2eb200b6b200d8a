export MOA_FFT_TF=2048
for lib in libmoa_fft libmoa_fft_m5 libmoa_fft_m6 libmoa_fft_t3; do
  for tma in 0 1; do
   echo "== $lib TMA=$tma"
   MOA_FFT_TMA=$tma MOA_FFT_LIB=$PWD/paper_0811_2535_b200/$lib.so timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
   MOA_FFT_TMA=$tma MOA_FFT_FUSE=0 MOA_FFT_LIB=$PWD/paper_0811_2535_b200/$lib.so timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
  done
done
