P="timeout 120 python tools/perf_probe.py"
for v in "" _A0; do
L=$PWD/paper_0811_2535_b200/libmoa_fft$v.so
echo "== $v"; MOA_FFT_LIB=$L MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
MOA_FFT_LIB=$L MOA_FFT_FUSE=2 MOA_FFT_DISCARD=0 $P 24 "256,256,256" 2>&1 | tail -1
MOA_FFT_LIB=$L MOA_FFT_FUSE=2 $P 26 "1024,256,256" 2>&1 | tail -1
done
MOA_FFT_LIB=$PWD/paper_0811_2535_b200/libmoa_fft_A0.so MOA_FFT_FUSE=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variant" 2>&1 | tail -2
