L=$PWD/paper_0811_2535_b200/libmoa_fft_R8.so
MOA_FFT_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lifted_all or explicit or variant or batched or 2d" 2>&1 | tail -2
P="timeout 120 python tools/perf_probe.py"
echo R16; $P 24 "256,256,256" 2>&1 | tail -1
echo R8; MOA_FFT_LIB=$L $P 24 "256,256,256" "64,512,512" "512,512,64" 2>&1 | grep '^{"t'
echo R8-fuse2; MOA_FFT_LIB=$L MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
echo R8-26; MOA_FFT_LIB=$L $P 26 "" 2>&1 | tail -1
echo R8-TF4096; MOA_FFT_LIB=$L MOA_FFT_TF=4096 $P 24 "256,256,256" 2>&1 | tail -1
