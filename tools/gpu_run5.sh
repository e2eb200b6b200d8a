for lib in libmoa_fft_old libmoa_fft_nohint libmoa_fft; do
  echo "== $lib"
  MOA_FFT_LIB=$PWD/paper_0811_2535_b200/$lib.so timeout 120 python tools/perf_probe.py 24 "4096,4096" "256,256,256" 2>&1 | tail -2
done
for lib in libmoa_fft_old libmoa_fft; do
MOA_FFT_LIB=$PWD/paper_0811_2535_b200/$lib.so timeout 120 python tools/perf_probe.py 24 "4096,4096" > gpurun_out/plain_$lib.log 2>&1 && MOA_FFT_LIB=$PWD/paper_0811_2535_b200/$lib.so ncu --set full --clock-control none -k regex:fft_pass -s 2 -c 1 -o gpurun_out/prof_$lib -f python tools/perf_probe.py 24 "4096,4096" > gpurun_out/ncu_$lib.log 2>&1
done
