P="timeout 120 python tools/perf_probe.py"
for tf in 4096 8192; do echo "TF=$tf"; MOA_FFT_TF=$tf $P 24 "4096,4096" "1024,16384" 2>&1 | grep '^{"t'; done
MOA_FFT_TF=2048 $P 24 "2048,8192" "1024,1024,16" 2>&1 | grep '^{"t'
MOA_FFT_TF=1024 $P 24 "1024,1024,16" 2>&1 | grep '^{"t'
