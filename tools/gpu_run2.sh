set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not slow" 2>&1 | tail -15
timeout 300 python tools/perf_probe.py 24 "" "256,256,256" "4096,4096" 2>&1 | tail -4
for sl in "2 1" "3 1" "3 2" "4 2"; do set -- $sl; MOA_FFT_SLOTS=$1 MOA_FFT_LAG=$2 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1; done
MOA_FFT_TF=2048 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
MOA_FFT_FUSE=0 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
for t in 20 21 22 23 25 26 27 28; do timeout 120 python tools/perf_probe.py $t "" 2>&1 | tail -1; done
timeout 300 python bench.py --steps 20 --warmup 3 2>&1 | tail -3
