for tf in 1024 2048 4096 8192; do echo "TF=$tf"; MOA_FFT_TF=$tf timeout 300 python tools/batch_probe.py 9x32768 10x16384 11x8192 12x4096 13x2048 2>&1 | grep '^{' | cut -c1-120; done
