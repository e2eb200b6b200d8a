"""SURVEY §8(f) N2 on the GPU: the layout redistributions of the paper (Fig 5.3 / 5.4 /
5.8 / 5.9) as library calls (moa_redist_*: CUDA pack/unpack kernels + the transfer
round), run on p virtual ranks of one B200 (MOA_MODE_EMULATED: the transfers become
device copies; real ranks use the same steps with NCCL -- tests/test_gpu_multi.py).

A redistribution moves data and computes nothing, so the bar is bit-exact equality
with the layouts written out by numpy slicing of the seeded input: BLOCK = x itself
(rank r's block at offset r*psize), CYCLIC = concat_r x[r::p], CENTRAL = x on rank 0.
Message counts are the paper's: m(m-1) for Fig 5.9's direct block <-> cyclic exchange
(P:1043), 2(m-1) through processor 0 (Fig 5.4), m-1 for a scatter / gather."""
import numpy as np
import pytest

import moa_inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_0811_2535_b200 as moa  # noqa: E402
from _parity import check  # noqa: E402

B, C, Z = moa.LAYOUT_BLOCK, moa.LAYOUT_CYCLIC, moa.LAYOUT_CENTRAL


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    moa.load()


def layout(x, p, kind):
    if kind == C:
        return np.concatenate([x[r::p] for r in range(p)])
    return x.copy()   # BLOCK (blocks back to back) and CENTRAL (rank 0's n) are x itself


CASES = [(B, C, moa.ROUTE_DIRECT), (C, B, moa.ROUTE_DIRECT), (B, C, moa.ROUTE_CENTRAL), (C, B, moa.ROUTE_CENTRAL),
         (Z, C, moa.ROUTE_DIRECT), (C, Z, moa.ROUTE_DIRECT), (Z, B, moa.ROUTE_DIRECT), (B, Z, moa.ROUTE_DIRECT),
         (C, C, moa.ROUTE_DIRECT), (B, B, moa.ROUTE_DIRECT)]


def expected_messages(p, frm, to, route):
    if frm == to:
        return 0
    if {frm, to} == {B, C}:
        return p * (p - 1) if route == moa.ROUTE_DIRECT else 2 * (p - 1)
    return p - 1


@pytest.mark.parametrize("t,p", [(2, 2), (6, 8), (10, 2), (12, 4), (16, 8), (17, 16), (22, 4), (24, 8)])
def test_redistributions_bit_exact(t, p):
    n = 1 << t
    x = moa_inputs.signal_for(t)
    for frm, to, route in CASES:
        plan = moa.Redist(n, p, frm, to, route, mode=moa.MODE_EMULATED)
        info = plan.info()
        assert info["messages"] == expected_messages(p, frm, to, route), (frm, to, route, info)
        got = plan.execute(torch.from_numpy(layout(x, p, frm)).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), layout(x, p, to)), (t, p, frm, to, route)
        plan.destroy()


def test_redistribution_bytes_and_bottleneck():
    """Fig 5.4's via-central route moves every element twice and loads processor 0's
    links with (p-1) psize each way; Fig 5.9's direct route sends psize (p-1)/p per rank
     -- the library's own counts."""
    n, p = 1 << 20, 8
    psize = n // p
    d = moa.Redist(n, p, B, C, moa.ROUTE_DIRECT, mode=moa.MODE_EMULATED).info()
    v = moa.Redist(n, p, B, C, moa.ROUTE_CENTRAL, mode=moa.MODE_EMULATED).info()
    assert d["max_rank_bytes"] == 16 * psize * (p - 1) // p
    assert v["max_rank_bytes"] == 16 * psize * (p - 1)


@pytest.mark.parametrize("t,p", [(12, 4), (20, 8), (24, 2)])
def test_block_natural_transform_emulated(t, p):
    """Block-natural input and output around the cyclic transform (two extra
    redistributions): BLOCK -> CYCLIC (direct), the partitioned FFT, CYCLIC -> BLOCK --
    rank r ends with X[r psize : (r+1) psize], i.e. the buffer equals the oracle's X."""
    n = 1 << t
    x = moa_inputs.signal_for(t)
    xd = torch.from_numpy(x).cuda()
    xc = moa.Redist(n, p, B, C, mode=moa.MODE_EMULATED).execute(xd)
    Xc = moa.Plan(n, p, -1, mode=moa.MODE_EMULATED).execute(xc)
    Xb = moa.Redist(n, p, C, B, mode=moa.MODE_EMULATED).execute(Xc)
    torch.cuda.synchronize()
    check(Xb.cpu().numpy(), oracle.fft(x, -1, threads=8), t, "block-natural transform (emulated p=%d)" % p)


def test_redist_rejections():
    with pytest.raises(moa.MoaError) as e:
        moa.Redist(6, 2, B, C, mode=moa.MODE_EMULATED)
    assert e.value.code == -1
    with pytest.raises(moa.MoaError) as e:
        moa.Redist(16, 8, B, C, mode=moa.MODE_EMULATED)   # psize < p
    assert e.value.code == -2
    with pytest.raises(moa.MoaError) as e:
        moa.Redist(1 << 10, 2, B, C)                       # real ranks without moa_dist_init
    assert e.value.code == -5
    plan = moa.Redist(1 << 10, 2, B, C, mode=moa.MODE_EMULATED)
    x = torch.zeros(1 << 10, dtype=torch.complex128, device="cuda")
    assert moa.load().moa_redist_execute(plan._h, x.data_ptr(), x.data_ptr()) == -9   # in place refused
