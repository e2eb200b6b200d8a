P="timeout 120 python tools/perf_probe.py"
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo pdl; MOA_FFT_PDL=1 $P 24 "256,256,256" 2>&1 | tail -1
echo pdl-22; MOA_FFT_PDL=1 $P 22 "" 2>&1 | tail -1
echo plain-22; $P 22 "" 2>&1 | tail -1
echo pdl-16; MOA_FFT_PDL=1 $P 16 "" 2>&1 | tail -1
echo plain-16; $P 16 "" 2>&1 | tail -1
echo pdl-28; MOA_FFT_PDL=1 $P 28 "" 2>&1 | tail -1
MOA_FFT_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lifted_all or explicit or inplace or large_sizes_full or batched or 2d" 2>&1 | tail -2
