P="timeout 300 python tools/perf_probe.py"
for o in 0 1 2 3; do echo "order=$o"; MOA_FFT_ORDER=$o $P 24 "" 2>&1 | tail -1 | cut -c1-400; MOA_FFT_ORDER=$o $P 26 "" 2>&1 | tail -1 | cut -c1-400; done
for o in 0 3; do MOA_FFT_ORDER=$o $P 28 "" 2>&1 | tail -1 | cut -c1-400; done
MOA_FFT_ORDER=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lifted_all or explicit or large_sizes_full or variant" 2>&1 | tail -2
