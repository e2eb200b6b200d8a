"""Host-side reference of the paper's layout redistributions over torch.distributed
(TEST INFRASTRUCTURE: exercised over gloo on the CPU by tests/test_dist_gloo.py).

These are the index maps of Fig 5.3/5.4/5.8/5.9 written with torch collectives; the
product calls (paper_0811_2535_b200.Redist and the functions built on it) implement the
same maps in CUDA pack kernels + NCCL and are checked against numpy slicing on the GPU
(tests/test_gpu_redist.py).
"""
def scatter_cyclic(x0, n: int, group=None, device=None):
    """The paper's DISTRIBUTE_CENTRALIZED_TO_CYCLIC_PARTITIONED (Fig 5.8):
    rank 0 holds the whole x0 (n elements); rank r receives xcyclic = x0[r::p] (psize
    elements).  Layout plumbing outside the transform (torch.distributed scatter);
    `device` is where the local slice lives (default: x0's device on rank 0, CPU
    elsewhere unless given)."""
    import torch
    import torch.distributed as dist
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    psize = n // p
    dev = device if device is not None else (x0.device if rank == 0 else torch.device("cpu"))
    mine = torch.empty(psize, dtype=torch.complex128, device=dev)
    chunks = None
    if rank == 0:
        chunks = [x0[r::p].contiguous().view(torch.float64).to(dev) for r in range(p)]
    out = mine.view(torch.float64)
    dist.scatter(out, chunks, src=0, group=group)
    return mine


def gather_cyclic(xcyclic, n: int, group=None):
    """The paper's DISTRIBUTE_CYCLIC_PARTITIONED_TO_CENTRALIZED (Fig 5.8):
    rank r holds X[r::p]; rank 0 returns the whole n-vector in natural order (x0(r:n-1:m)
    = xcyclic of rank r), the other ranks return None."""
    import torch
    import torch.distributed as dist
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    psize = n // p
    flat = xcyclic.contiguous().view(torch.float64)
    parts = [torch.empty_like(flat) for _ in range(p)] if rank == 0 else None
    dist.gather(flat, parts, dst=0, group=group)
    if rank != 0:
        return None
    x0 = torch.empty(n, dtype=torch.complex128, device=xcyclic.device)
    for r in range(p):
        x0[r::p] = parts[r].view(torch.complex128)[:psize]
    return x0


def block_to_cyclic(x_block, group=None):
    """Fig 5.3 / Fig 5.9's direct redistribution applied to the INPUT: rank r
    holds the natural block x[r*psize : (r+1)*psize] and gets xcyclic = x[r::p] -- one
    all-to-all (m(m-1) messages of psize/m): element i of block r goes to rank i mod p,
    slot r*psize/p + i div p.  Layout plumbing over torch.distributed, outside the
    transform (block-natural in/out costs two extra all-to-alls)."""
    import torch
    import torch.distributed as dist
    p = dist.get_world_size(group)
    m = x_block.numel()
    send = x_block.contiguous().view(m // p, p).t().contiguous()        # [dst][q]: x[r*psize + dst + p*q]
    recv = torch.empty(2 * m, dtype=torch.float64, device=x_block.device)
    dist.all_to_all_single(recv, send.view(torch.float64).reshape(-1), group=group)
    return recv.view(torch.complex128)                                  # [src r][q] = x[rank + p*(r*psize/p + q)]


def cyclic_to_block(x_cyclic, group=None):
    """The inverse redistribution for the OUTPUT: rank d holds X[d + p*i'] (the transform's
    xcyclic) and gets the natural block X[d*psize : (d+1)*psize] -- chunk r of the cyclic
    slice (i' in [r*psize/p, (r+1)*psize/p)) goes to rank r, which interleaves the p
    chunks it receives (element q of source d lands at d + p*q)."""
    import torch
    import torch.distributed as dist
    p = dist.get_world_size(group)
    m = x_cyclic.numel()
    recv = torch.empty(2 * m, dtype=torch.float64, device=x_cyclic.device)
    dist.all_to_all_single(recv, x_cyclic.contiguous().view(torch.float64), group=group)
    return recv.view(torch.complex128).view(p, m // p).t().reshape(-1)


def block_to_cyclic_via_central(x_block, group=None):
    """Fig 5.4: the same redistribution routed through processor 0 --
    every block is sent to rank 0 (m-1 messages of psize), which sends every rank its
    cyclic slice (m-1 messages of psize): 2(m-1) messages, each element moved twice,
    rank 0's links the bottleneck.  The ablation of Fig 5.9's direct exchange."""
    import torch
    import torch.distributed as dist
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    m = x_block.numel()
    flat = x_block.contiguous().view(torch.float64)
    parts = [torch.empty_like(flat) for _ in range(p)] if rank == 0 else None
    dist.gather(flat, parts, dst=0, group=group)                        # x0 on processor 0
    mine = torch.empty(2 * m, dtype=torch.float64, device=x_block.device)
    chunks = None
    if rank == 0:
        x0 = torch.cat([q.view(torch.complex128) for q in parts])
        chunks = [x0[r::p].contiguous().view(torch.float64) for r in range(p)]
    dist.scatter(mine, chunks, src=0, group=group)                      # xcyclic from processor 0
    return mine.view(torch.complex128)
