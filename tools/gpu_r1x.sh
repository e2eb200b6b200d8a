timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py > gpurun_out/bench_x.log 2>&1; grep '^{' gpurun_out/bench_x.log | tail -1 | cut -c1-700
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 2>&1 | grep '^{' | cut -c1-400
