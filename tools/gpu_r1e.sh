P="timeout 120 python tools/perf_probe.py"
L5=$PWD/paper_0811_2535_b200/libmoa_fft_m5.so
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo plain-m5; MOA_FFT_LIB=$L5 $P 24 "256,256,256" 2>&1 | tail -1
echo fuse2-m5; MOA_FFT_LIB=$L5 MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
echo fuse2-T16; MOA_FFT_FUSE=2 MOA_FFT_TF=4096 $P 24 "256,256,256" 2>&1 | tail -1
echo plain-26-m5; MOA_FFT_LIB=$L5 $P 26 "1024,256,256" 2>&1 | tail -1
