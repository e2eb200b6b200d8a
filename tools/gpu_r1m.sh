timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python tools/sweep.py --tmin 4 --tmax 30 --md gpurun_out/sweep.md > gpurun_out/sweep.log 2>&1; tail -3 gpurun_out/sweep.log
timeout 300 python bench.py > gpurun_out/bench_m.log 2>&1; tail -c 600 gpurun_out/bench_m.log
