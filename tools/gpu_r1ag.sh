timeout 600 python tools/dist_model.py --t 24 26 --md gpurun_out/dist_model.md 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "plan_info or large_sizes or lifted_all" 2>&1 | tail -2
