timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "batched or lifted_all or plan_info or emulated" 2>&1 | tail -3
timeout 300 python tools/batch_probe.py 10x16384 12x4096 13x2048 16x256 20x16 4x1048576 8x65536
