timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "nd_ or 2d or 3d" 2>&1 | tail -3
