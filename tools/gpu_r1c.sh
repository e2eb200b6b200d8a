timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variant" 2>&1 | tail -3
timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
for sl in "4 2" "3 1" "6 3" "8 4" "5 2"; do set -- $sl; echo "slots=$1 lag=$2"; MOA_FFT_FUSE=2 MOA_FFT_SLOTS=$1 MOA_FFT_LAG=$2 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1; done
MOA_FFT_FUSE=2 MOA_FFT_DISCARD=0 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
MOA_FFT_FUSE=2 timeout 120 python tools/perf_probe.py 24 "512,256,128" 2>&1 | tail -1
MOA_FFT_FUSE=2 timeout 120 python tools/perf_probe.py 24 "128,256,512" 2>&1 | tail -1
MOA_FFT_FUSE=2 timeout 120 python tools/perf_probe.py 22 "64,256,256" 2>&1 | tail -1
MOA_FFT_FUSE=2 timeout 120 python tools/perf_probe.py 23 "128,256,256" 2>&1 | tail -1
MOA_FFT_FUSE=2 timeout 120 python tools/perf_probe.py 20 "16,256,256" 2>&1 | tail -1
MOA_FFT_FUSE=2 timeout 120 python tools/perf_probe.py 24 "256,256,256" > gpurun_out/f2plain.log 2>&1 && MOA_FFT_FUSE=2 ncu --set full --import-source on --clock-control none -k regex:"fused" -s 1 -c 1 -o gpurun_out/prof_f2 -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu_f2.log 2>&1; tail -2 gpurun_out/ncu_f2.log
