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


# --------------------------------------------------------------- K11: global re-blocking
# Per-shard positions columns are canonical columns of their own row ranges (D-18),
# but their blocks are aligned to each shard's own output ranks. K11 (SURVEY.md
# §8(e), §8(f) #4) re-blocks them into ONE global DELTA_BP{B} column distributed
# over the ranks: global block k (output ranks [kB, kB + B)) is owned by the rank
# holding rank kB + B - 1; a rank receives the head of its first owned block from
# the predecessors' tails (each rank's last < B positions, one allgather of
# world x B u64 plus the counts) and the cw offset of its first block (one more
# allgather of 8-byte width totals); the last rank holds the final partial block
# (the remainder). Blocks are independent (D-6), so a rank's blocks are
# byte-identical to the same blocks of the single-column image.

def reblock_contribution(pos, B: int = 512):
    """Phase 1 on every rank: (count, tail) with tail = this shard's last
    min(n, B - 1) positions as a device int64 tensor padded to B - 1."""
    from paper_2004_09350_b200 import ms
    n = pos.n
    vals = ms.decompress(pos)
    L = min(n, B - 1)
    tail = torch.zeros(B - 1, dtype=torch.int64, device=vals.device)
    if L:
        tail[:L] = vals[n - L:]
    return n, tail, vals


def reblock_local(vals, rank: int, counts: list[int], tails: list, B: int = 512):
    """Phase 2: this rank's blocks of the global column as a DELTA_BP{B} column
    (cw local from 0; the last rank's column carries the global remainder), and
    the global index of its first block."""
    from paper_2004_09350_b200 import ms
    world = len(counts)
    O = sum(counts[:rank])
    N = sum(counts)
    n = counts[rank]
    ka, kb = O // B, (O + n) // B
    h = O - ka * B
    last = rank == world - 1
    parts = []
    if h and (kb > ka or last):  # head: ranks [ka B, O) from the predecessors' tails, newest first
        need, pieces = h, []
        for r in range(rank - 1, -1, -1):
            if not need:
                break
            c = counts[r]
            take = min(c, need)
            if take:
                Lr = min(c, B - 1)
                pieces.append(tails[r][Lr - take:Lr])
                need -= take
        if need:
            raise RuntimeError("reblock: fewer preceding positions than the head needs")
        parts.extend(reversed(pieces))
    own_end = (kb * B - O) if kb * B >= O else 0
    if last:
        parts.append(vals)  # everything: full blocks and the remainder
    elif kb > ka:
        parts.append(vals[:own_end])
    seq = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.int64, device=vals.device)
    if not last:
        assert seq.numel() == (kb - ka) * B
    col = ms.compress(seq, ms.delta_bp(B))
    return col, ka


def reblock_positions(pos, B: int = 512, device=None):
    """K11 under torch.distributed: this rank's slice of the globally re-blocked
    DELTA_BP{B} column. Returns (column with local cw, first global block, global
    cw offset of that block)."""
    n, tail, vals = reblock_contribution(pos, B)
    world = dist.get_world_size()
    cnt = torch.tensor([n], dtype=torch.int64, device=tail.device)
    counts_t = torch.empty(world, dtype=torch.int64, device=tail.device)
    dist.all_gather_into_tensor(counts_t, cnt)
    tails_t = torch.empty(world * (B - 1), dtype=torch.int64, device=tail.device)
    dist.all_gather_into_tensor(tails_t, tail)
    counts = counts_t.tolist()
    tails = list(tails_t.view(world, B - 1))
    col, ka = reblock_local(vals, dist.get_rank(), counts, tails, B)
    wsum = torch.tensor([col.payload_words * 64 // B], dtype=torch.int64, device=tail.device)
    wall = torch.empty(world, dtype=torch.int64, device=tail.device)
    dist.all_gather_into_tensor(wall, wsum)
    return col, ka, int(sum(wall.tolist()[:dist.get_rank()]))
