timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/sweep.py --tmin 4 --tmax 30 --md gpurun_out/sweep2.md > gpurun_out/sweep2.log 2>&1; tail -2 gpurun_out/sweep2.log
