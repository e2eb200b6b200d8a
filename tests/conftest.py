import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def read_golden(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([c.strip() for c in line.split("|")])
    return rows


def parse_complex_list(s):
    out = []
    for tok in s.split():
        re_, im_ = tok.split(",")
        out.append(complex(float(re_), float(im_)))
    return out


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print the achieved relL2 of every recorded GPU parity check against its bar."""
    try:
        import _parity
    except Exception:
        return
    recs = _parity.RECORDS
    if not recs:
        return
    tr = terminalreporter
    tr.section("achieved relL2 (GPU vs oracle; bar = 1e-12 log2 n)")
    worst = {}
    for r in recs:
        k = (r["test"], r["t"])
        if k not in worst or r["relL2"] > worst[k]["relL2"]:
            worst[k] = r
    for (name, t), r in sorted(worst.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        tr.write_line(f"t={t:2d}  relL2={r['relL2']:.3e}  bar={r['bar']:.1e}  margin={r['bar'] / max(r['relL2'], 1e-300):9.0f}x  {name}")
    out = os.environ.get("MOA_PARITY_LOG")
    if out:
        _parity.dump(out)
