set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_a.log 2>&1; tail -c 3000 gpurun_out/bench_a.log
for spec in "256,256,256" "4096,4096" "2048,8192" "8192,2048" "64,512,512" "512,512,64"; do
  timeout 120 python tools/perf_probe.py 24 "$spec" 2>&1 | tail -1
done
MOA_FFT_FUSE=1 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
MOA_FFT_FUSE=1 MOA_FFT_TF=2048 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
for t in 20 22 26 28; do timeout 120 python tools/perf_probe.py $t "" 2>&1 | tail -1; done
