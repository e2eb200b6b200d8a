set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -30
for tf in 8192 4096; do MOA_FFT_TF=$tf timeout 300 python tools/perf_probe.py 24 "4096,4096" "2048,8192" "8192,2048" "256,256,256" 2>&1 | tail -8; done
timeout 300 python tools/perf_probe.py 20 "" 2>&1 | tail -3
timeout 300 python tools/perf_probe.py 22 "" 2>&1 | tail -3
