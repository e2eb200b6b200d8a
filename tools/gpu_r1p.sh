P="timeout 120 python tools/perf_probe.py"
for tf in 2048 1024 512 256; do echo "TF=$tf"; MOA_FFT_TF=$tf $P 24 "256,256,256" 2>&1 | tail -1; done
for tf in 1024 512; do echo "TF=$tf fuse2"; MOA_FFT_TF=$tf MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1; done
for tf in 1024 512; do echo "TF=$tf t26"; MOA_FFT_TF=$tf $P 26 "256,256,1024" 2>&1 | tail -1; done
