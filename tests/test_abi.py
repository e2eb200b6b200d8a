"""CPU-side checks of the C-ABI boundary: the library builds, loads, exports
every symbol include/moa_fft.h declares, and validates its arguments (naming
the violated bound) before it touches a GPU."""
import ctypes
import os
import re

import pytest

import paper_0811_2535_b200 as moa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", fn)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(moa_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("moa_fft_plan", "moa_fft_execute", "moa_fft_destroy", "moa_fft_set_stream",
                     "moa_dist_init", "moa_dist_finalize", "moa_fft_plan_info", "moa_fft_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = moa.load()
    missing = [n for n in _declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(moa.EXPORTS) <= set(_declared_functions())
    assert b"sm_100a" in lib.moa_fft_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", moa.lib_path()], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("n,p,sign,code,needle", [
    (6, 1, -1, -1, "2^t"),
    (1, 1, -1, -1, "2^t"),
    (0, 1, -1, -1, "2^t"),
    (1 << 33, 1, -1, -1, "t <= 32"),
    (16, 1, 0, -3, "sign"),
    (16, 3, -1, -2, "power of two"),
    (16, 8, -1, -2, "psize >= m"),     # n=16, m=8 rejected
])
def test_plan_validation_errors(n, p, sign, code, needle):
    lib = moa.load()
    h = lib.moa_fft_plan(n, p, sign)
    assert not h
    msg = lib.moa_fft_last_error().decode()
    assert needle in msg, msg
    assert lib.moa_fft_last_error_code() == code   # the code that goes with the message
    with pytest.raises(moa.MoaError) as e:
        moa.Plan(n, p, sign)
    assert e.value.code == code   # Plan() raises the library's own MOA_ERR_* code
    assert needle in str(e.value)


def test_last_error_code_tracks_the_last_failure():
    lib = moa.load()
    assert not lib.moa_fft_plan(6, 1, -1)
    assert lib.moa_fft_last_error_code() == -1          # INVALID_N (Fig 2.1: n = 2^t)
    assert not lib.moa_fft_plan(16, 1, 2)
    assert lib.moa_fft_last_error_code() == -3          # INVALID_SIGN
    assert lib.moa_fft_execute(None, None, None) == -9
    assert lib.moa_fft_last_error_code() == -9          # INVALID_ARG (NULL plan)


def test_product_library_holds_only_adopted_kernels():
    """The variants measured slower (persistent / TMA-staged / prefetching
    passes, the L2-fused pass pair) are compiled only into libmoa_fft_variants.so."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "-sass", moa.lib_path()], capture_output=True, text=True)
    assert out.returncode == 0
    names = re.findall(r"Function : (\S+)", out.stdout)
    assert names
    banned = ("fft_pass_tma_kernel", "fft_pass_tpf_kernel", "fft_pass_pf_kernel", "fft_pass_rdb_kernel",
              "fft_pass_persist_kernel", "fused_kernel", "fused_ticket_kernel")
    bad = [nm for nm in names if any(b in nm for b in banned)]
    assert not bad, bad[:5]


def test_execute_rejects_null_plan():
    lib = moa.load()
    assert lib.moa_fft_execute(None, None, None) == -9
    assert lib.moa_fft_plan_info(None, None) == -9
    lib.moa_fft_destroy(None)  # NULL-safe


def test_dist_plan_without_init_is_rejected():
    lib = moa.load()
    h = lib.moa_fft_plan(1 << 10, 2, -1)
    assert not h
    assert "moa_dist_init" in lib.moa_fft_last_error().decode()


@pytest.mark.parametrize("kw,needle", [
    ({"p": 2, "batch": 4, "mode": moa.MODE_EMULATED}, "batch > 1 needs p == 1"),
    ({"batch": 4, "mode": moa.MODE_LITERAL}, "batch > 1 needs p == 1"),
    ({"batch": -3}, "batch -3 < 0"),
    ({"p": 2, "exchange": 7, "mode": moa.MODE_EMULATED}, "unknown exchange"),
    ({"p": 2, "exchange": moa.XCHG_P2P_EXTERNAL, "rank": 5}, "rank 5 outside"),
])
def test_option_validation_errors(kw, needle):
    """Option checks run before any device call (CPU-testable)."""
    p = kw.pop("p", 1)
    with pytest.raises(moa.MoaError) as e:
        moa.Plan(1 << 10, p, -1, **kw)
    assert needle in str(e.value), str(e.value)


def test_p2p_calls_reject_non_p2p_plans():
    lib = moa.load()
    assert lib.moa_fft_ipc_handle(None, None) == -9
    assert lib.moa_fft_ipc_open(None, None) == -9
    assert lib.moa_fft_enable_p2p(None) == -9
    assert lib.moa_fft_execute_phase(None, None, None, 1) == -9
    assert lib.moa_fft_execute_host_batch(None, 0, None, None) == -9


@pytest.mark.parametrize("shape,needle", [
    ((4,), "rank 1 must be 2 or 3"),
    ((2, 2, 2, 2), "rank 4 must be 2 or 3"),
    ((3, 8), "n1=3 must be 2^t"),
    ((1 << 27, 4), "<= 26"),
    ((8, 6), "n2=6 must be 2^t"),
    ((1 << 16, 1 << 17), "more than 2^32"),
])
def test_nd_plan_validation_errors(shape, needle):
    """r-D plan checks run before any device call (CPU-testable)."""
    with pytest.raises(moa.MoaError) as e:
        moa.PlanND(shape)
    assert needle in str(e.value), str(e.value)


def test_binding_structs_match_the_header_layout(tmp_path):
    """The ctypes mirrors of moa_fft_options / moa_fft_info / moa_fft_kernel_stat have the
    size and field offsets the C compiler gives the header's structs (an ABI drift check:
    a field added on one side only would shift every later field)."""
    fields = {"moa_fft_options": moa._Options, "moa_fft_info": moa._Info, "moa_fft_kernel_stat": moa._KernelStat}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "moa_fft.h"', "int main(void) {"]
    for cname, py in fields.items():
        lines.append(f'    printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'    printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["    return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    import subprocess
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", str(src), "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in fields.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_c_client_compiles_links_and_runs(tmp_path):
    """The header is a C99 header and the library links from plain C: gcc builds
    tests/c/abi_host.c against include/moa_fft.h and libmoa_fft.so, and its host-only
    checks (default lifting, a pass's index map, error codes + messages) pass on the CPU."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not on PATH")
    moa.load()
    exe = str(tmp_path / "abi_host")
    libdir = os.path.dirname(moa.lib_path())
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c", "abi_host.c"), "-o", exe, moa.lib_path(),
                        f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


@pytest.mark.parametrize("n,p,frm,to,route,mode,code,needle", [
    (6, 2, 0, 1, 0, 2, -1, "2^t"),                 # n not a power of two (Fig 2.1)
    (1 << 10, 3, 0, 1, 0, 2, -2, "power of two"),
    (16, 8, 0, 1, 0, 2, -2, "psize"),              # psize < m
    (1 << 10, 2, 0, 3, 0, 2, -9, "layout"),        # unknown layout
    (1 << 10, 2, 0, 1, 2, 2, -9, "route"),         # unknown route
    (1 << 10, 2, 0, 1, 0, 1, -9, "mode"),          # MOA_MODE_LITERAL is not a redistribution mode
    (1 << 10, 2, 0, 1, 0, 0, -5, "moa_dist_init"), # real ranks without the communicator
])
def test_redist_plan_validation(n, p, frm, to, route, mode, code, needle):
    """moa_redist_plan validates before it touches a GPU: NULL plus the
    code and a message naming the violated bound."""
    lib = moa.load()
    assert not lib.moa_redist_plan(n, p, frm, to, route, mode)
    assert lib.moa_fft_last_error_code() == code
    assert needle in lib.moa_fft_last_error().decode()
    assert lib.moa_redist_execute(None, None, None) == -9
    lib.moa_redist_destroy(None)   # NULL-safe
