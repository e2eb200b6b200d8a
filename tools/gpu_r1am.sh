P="timeout 120 python tools/perf_probe.py"
for t in 17 18 19 20 21 22 23; do $P $t "" 2>&1 | tail -1 | cut -c1-150; MOA_FFT_TMA=2 $P $t "" 2>&1 | tail -1 | cut -c1-150; done
