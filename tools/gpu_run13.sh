timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not slow" 2>&1 | tail -3
export MOA_FFT_TF=2048
for tma in 1 0; do
   echo "TMA=$tma"
   MOA_FFT_TMA=$tma timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
   MOA_FFT_TMA=$tma MOA_FFT_FUSE=0 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
done
for sl in "6 3" "8 4" "10 6" "12 8"; do set -- $sl; echo "slots $1 lag $2"; MOA_FFT_SLOTS=$1 MOA_FFT_LAG=$2 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1; done
