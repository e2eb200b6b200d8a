"""The GPU parity bar and a record of the achieved errors (test infrastructure).

check(got, ref, t, name): relL2 = ||g - o|| / ||o|| accumulated in long double
(oracle.rel_l2) must be <= 1e-12 * log2 n (BASELINE.json
north_star).  Every check is recorded; tests/conftest.py prints the table of achieved
relL2 against the bar at the end of the session (the margin is visible in the log).
"""
import json
import os

import numpy as np

import oracle

RECORDS = []


def bar(t: int) -> float:
    return 1e-12 * t


def record(name: str, t: int, err: float):
    RECORDS.append({"test": name, "t": int(t), "relL2": float(err), "bar": bar(t)})


def check(got, ref, t: int, name: str) -> float:
    err = oracle.rel_l2(got, ref)
    record(name, t, err)
    assert err <= bar(t), f"{name}: relL2 {err:.3e} > {bar(t):.1e} (t={t})"
    return err


def check_parts(num, den, t: int, name: str) -> float:
    """the same bar from accumulated (sum |g-o|^2, sum |o|^2) parts (chunked comparisons)"""
    err = float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))
    record(name, t, err)
    assert err <= bar(t), f"{name}: relL2 {err:.3e} > {bar(t):.1e} (t={t})"
    return err


def parts_threads(got, ref, chunk: int = 1 << 24, threads: int = 0):
    """oracle.l2_parts over chunks on a thread pool (same long-double sums, regrouped by
    chunk): for 2^27..2^31-element comparisons.  got/ref: equal-length 1-D arrays (views)."""
    from concurrent.futures import ThreadPoolExecutor
    n = len(ref)
    assert len(got) == n
    with ThreadPoolExecutor(threads or len(os.sched_getaffinity(0))) as ex:
        parts = list(ex.map(lambda s: oracle.l2_parts(got[s:s + chunk], ref[s:s + chunk]), range(0, n, chunk)))
    return sum(p[0] for p in parts), sum(p[1] for p in parts)


def dump(path: str):
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(RECORDS, f, indent=0)
