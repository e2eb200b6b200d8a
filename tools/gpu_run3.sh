set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not slow" 2>&1 | tail -5
timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_DISCARD=0 timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_SCRST=0 timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_P2LD=0 MOA_FFT_P3ST=0 timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_LDHINT=0 timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_SLOTS=4 MOA_FFT_LAG=2 timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_TF=2048 timeout 300 python tools/perf_probe.py 24 "" 2>&1 | tail -1
MOA_FFT_FUSE=0 timeout 300 python tools/perf_probe.py 24 "256,256,256" "4096,4096" 2>&1 | tail -2
MOA_FFT_FUSE=0 MOA_FFT_LDHINT=0 timeout 300 python tools/perf_probe.py 24 "256,256,256" "4096,4096" 2>&1 | tail -2
timeout 300 python tools/perf_probe.py 24 "" > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -o gpurun_out/prof_fused -f python tools/perf_probe.py 24 "" > gpurun_out/ncu_fused.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fft_pass -c 1 -o gpurun_out/prof_pass0 -f python tools/perf_probe.py 24 "" > gpurun_out/ncu_pass0.log 2>&1
