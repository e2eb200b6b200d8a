P="timeout 120 python tools/perf_probe.py"
for v in "" _NA; do L=$PWD/paper_0811_2535_b200/libmoa_fft$v.so; echo "== $v"; MOA_FFT_LIB=$L $P 24 "256,256,256" 2>&1 | tail -1; MOA_FFT_LIB=$L $P 26 "" 2>&1 | tail -1; MOA_FFT_LIB=$L MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1; done
