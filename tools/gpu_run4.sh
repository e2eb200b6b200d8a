for lib in libmoa_fft_old libmoa_fft_nohint libmoa_fft libmoa_fft_old libmoa_fft_nohint libmoa_fft; do
  echo "== $lib"
  MOA_FFT_LIB=$PWD/paper_0811_2535_b200/$lib.so timeout 120 python tools/perf_probe.py 24 "256,256,256" "4096,4096" 2>&1 | tail -2
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
