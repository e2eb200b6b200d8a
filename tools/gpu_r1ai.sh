timeout 120 python tools/pcie_probe.py
P="timeout 120 python tools/perf_probe.py"
$P 24 literal 2>&1 | tail -1 | cut -c1-200
$P 20 literal 2>&1 | tail -1 | cut -c1-200
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
