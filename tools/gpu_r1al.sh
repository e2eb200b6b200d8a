MOA_FFT_TMA=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variant or lifted_all or explicit or large_sizes_full" 2>&1 | tail -2
P="timeout 120 python tools/perf_probe.py"
echo plain; $P 24 "256,256,256" 2>&1 | tail -1
echo tpf; MOA_FFT_TMA=2 $P 24 "256,256,256" 2>&1 | tail -1
echo tpf-26; MOA_FFT_TMA=2 $P 26 "" 2>&1 | tail -1
echo tpf-22; MOA_FFT_TMA=2 $P 22 "" 2>&1 | tail -1
MOA_FFT_TMA=2 $P 24 "256,256,256" > gpurun_out/tpf_plain.log 2>&1 && MOA_FFT_TMA=2 ncu --set full --import-source on --clock-control none -k regex:"tpf" -s 3 -c 3 -o gpurun_out/prof_tpf -f python tools/perf_probe.py 24 "256,256,256" > gpurun_out/ncu_tpf.log 2>&1; tail -1 gpurun_out/ncu_tpf.log
