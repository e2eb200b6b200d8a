#!/bin/bash
# Multi-GPU evidence in one go: run on a box
# with >= 8 B200s from the repo root.  Every gpurun call of this build had one GPU, so none
# of this has run yet; the outputs land in gpurun_out/multi_*.
set -x
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
# 1. real-rank parity of every exchange (NCCL chunked / unchunked, fused NVLink push, low end),
#    N2 redistributions and dist_fft_block, for p = 2, 4, 8 (skips what the box cannot host)
python -m pytest tests/test_gpu_multi.py -q > gpurun_out/multi_pytest.log 2>&1
# 2. the scaling lines: strong scaling of 2^24 (and 2^26) with the default (auto) exchange and
#    with NCCL forced; each line carries the no-overlap a2a block (busBw vs 900/770 GB/s,
#    fused-push extra time, overlap efficiency)
for p in 1 2 4 8; do
  [ "$p" -le "$N" ] || continue
  for t in 24 26; do
    python bench.py --gpus $p --t $t --steps 20 --warmup 5 --no-e2e > gpurun_out/multi_bench_p${p}_t${t}.json 2> gpurun_out/multi_bench_p${p}_t${t}.err
    [ "$p" -gt 1 ] && python bench.py --gpus $p --t $t --steps 20 --warmup 5 --no-e2e --exchange nccl \
        > gpurun_out/multi_bench_p${p}_t${t}_nccl.json 2> gpurun_out/multi_bench_p${p}_t${t}_nccl.err
  done
done
# 3. N2 on NVSwitch: Fig 5.9 direct vs Fig 5.4 via processor 0, real ranks
for p in 2 4 8; do
  [ "$p" -le "$N" ] || continue
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$p --master-addr=127.0.0.1 --master-port=$((29600 + p)) \
      tools/redist_probe.py 24 > gpurun_out/multi_redist_p$p.jsonl 2> gpurun_out/multi_redist_p$p.err
done
# 4. NVLink bytes of the fused push pass on one rank of a 2-rank P2P_EXTERNAL run (ncu attaches
#    to a single process; the push pass should move 16 M (p-1)/p bytes): see DESIGN.md §6
echo done
