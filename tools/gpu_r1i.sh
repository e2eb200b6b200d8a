timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
P="timeout 120 python tools/perf_probe.py"
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo tma; MOA_FFT_TMA=1 $P 24 "256,256,256" 2>&1 | tail -1
echo fuse1; MOA_FFT_FUSE=1 $P 24 "256,256,256" 2>&1 | tail -1
echo tma-fuse1; MOA_FFT_TMA=1 MOA_FFT_FUSE=1 $P 24 "256,256,256" 2>&1 | tail -1
echo fuse2; MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
echo tma-26; MOA_FFT_TMA=1 $P 26 "" 2>&1 | tail -1
