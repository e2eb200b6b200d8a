timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variant or lifted_all" 2>&1 | tail -3
MOA_FFT_PF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lifted_all or explicit or large_sizes_full" 2>&1 | tail -3
P="timeout 120 python tools/perf_probe.py"
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo pf; MOA_FFT_PF=1 $P 24 "256,256,256" 2>&1 | tail -1
echo pf-fuse2; MOA_FFT_PF=1 MOA_FFT_FUSE=2 $P 24 "256,256,256" 2>&1 | tail -1
echo pf-26; MOA_FFT_PF=1 $P 26 "" "64,16,256,256" 2>&1 | tail -2
echo pf-22; MOA_FFT_PF=1 $P 22 "" 2>&1 | tail -1
MOA_FFT_PF=1 $P 24 "256,256,256" > gpurun_out/pfplain.log 2>&1 && MOA_FFT_PF=1 ncu --set full --import-source on --clock-control none -k regex:"fft_pass" -s 3 -c 1 -o gpurun_out/prof_pf -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu_pf.log 2>&1; tail -1 gpurun_out/ncu_pf.log
