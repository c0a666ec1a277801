"""Single-box partitioning by row range and the cross-GPU combine step
(BASELINE.json configs[4]).

Each GPU owns a contiguous, 2048-row-aligned row range; 2048 is a multiple of
every block size (and of 64), so every shard is a canonical column on its own
and no block crosses a shard boundary. select runs with row_offset = the
shard's first row, so positions are global row ids (D-10). The only exchange
steps are:
  C1  allgather(count_s) -> exclusive scan -> each shard's output-index offset
  C2  allreduce(sum) of the per-shard sums (uint64 wrap-around == int64
      two's-complement addition, so an int64 NCCL/gloo sum is exact mod 2^64)
Both are 8-byte messages: latency-bound, on the compute stream.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ALIGN = 2048


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[start, end) of rank's rows: start_s = floor(s*n / (G*2048)) * 2048 (end_G = n)."""
    def start(s):
        return n if s >= world else (s * n // (world * ALIGN)) * ALIGN
    return start(rank), start(rank + 1)


def allgather_counts(count: int, device) -> list[int]:
    """C1: every rank's selected count (one int64 per rank)."""
    world = dist.get_world_size()
    t = torch.tensor([count], dtype=torch.int64, device=device)
    out = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t)
    return out.tolist()  # one device -> host read for all ranks


def exclusive_offsets(counts: list[int]) -> list[int]:
    offs, acc = [], 0
    for c in counts:
        offs.append(acc)
        acc += c
    return offs


def allreduce_u64_sum(t: torch.Tensor) -> torch.Tensor:
    """C2: in-place sum of a 1-element int64 tensor holding uint64 bits (mod 2^64)."""
    assert t.dtype == torch.int64
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
