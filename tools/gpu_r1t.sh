P="timeout 120 python tools/perf_probe.py"
for st in 0 400 800 1600 3000; do echo "stagger=$st"; MOA_FFT_STAGGER=$st $P 24 "256,256,256" 2>&1 | tail -1; done
for st in 800 1600; do echo "stagger=$st fuse2"; MOA_FFT_STAGGER=$st MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1; done
