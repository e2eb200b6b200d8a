"""Multi-GPU parity: the partitioned transform with REAL
ranks, one process per B200 over NCCL -- the NCCL all-to-all (unchunked and chunked),
the fused NVLink push, the low-end breakpoint and dist_fft -- each rank's X[r + P i]
against the oracle.  Needs P GPUs on the box: skipped where fewer are visible (every
gpurun call of this build gets one B200; the emulated and IPC tests cover the same data
path on one GPU)."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,ts", [(2, [12, 20, 24]), (4, [12, 20, 24]), (8, [12, 20, 24])])
def test_multi_gpu_partitioned_transform(world, ts):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs, {_ngpus()} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "dist_worker.py"),
           *[str(t) for t in ts]]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and "ALL-OK" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bench_multi_gpu_line(world):
    """bench.py --gpus N launches N ranks itself and reports n_gpus == gpus_active == N."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs, {_ngpus()} visible")
    import json
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--steps", "3",
                        "--warmup", "3", "--no-cpu", "--no-e2e", "--t", "20"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world and line["gpus_active"] == world
    assert "a2a" in line and "error" not in line["a2a"]
