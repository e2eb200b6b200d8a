timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not slow" 2>&1 | tail -3
for tf in 4096 2048; do
 for tma in 1 0; do
  echo "TF=$tf TMA=$tma"
  MOA_FFT_TF=$tf MOA_FFT_TMA=$tma timeout 120 python tools/perf_probe.py 24 "256,256,256" "4096,4096" 2>&1 | tail -3
  MOA_FFT_TF=$tf MOA_FFT_TMA=$tma MOA_FFT_FUSE=0 timeout 120 python tools/perf_probe.py 24 "256,256,256" 2>&1 | tail -1
 done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
