timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "3d or 2d" 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/bench_y.log 2>&1; grep '^{' gpurun_out/bench_y.log | tail -1 > gpurun_out/bench_y.json; cut -c1-400 gpurun_out/bench_y.json
