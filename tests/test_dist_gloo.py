"""Multi-process (world size 2, gloo, CPU) tests of the N>1 host logic of the
sharded path: row-range shards, C1 allgather
of the per-shard counts -> exclusive output offsets, C2 allreduce of the
per-shard sums mod 2^64. Each rank computes its shard with the ORACLE (no GPU
here); the assembled result must equal the single-column oracle (D-18)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2004_09350_b200 import dist as D

N = (1 << 16) + 2048 * 3 + 100  # ragged: the last shard carries a block remainder
SEL = 1 << 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, end = D.shard_range(N, world, rank)
        x = synth.gen_host("c5.X", end - start, start)
        y = synth.gen_host("c5.Y", end - start, start)
        X = O.encode(x, O.DYN_BP, 0, 512)
        Y = O.encode(y, O.FOR_BP, 0, 512)
        pos = O.select(X, O.LT, SEL, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
        yp = O.project(Y, pos, start, O.FOR_BP, 0, 512)
        counts = D.allgather_counts(pos.n, "cpu")
        offs = D.exclusive_offsets(counts)
        s = torch.tensor([O.agg_sum(yp)], dtype=torch.uint64).view(torch.int64)
        D.allreduce_u64_sum(s)
        # wrap-around: every rank contributes 2^63 -> 0 mod 2^64 for an even world
        w = torch.tensor([1 << 63], dtype=torch.uint64).view(torch.int64)
        D.allreduce_u64_sum(w)
        mx = D.max_over_ranks(float(rank + 1), "cpu")
        q.put((rank, start, end, counts, offs, O.decode(pos).tolist(), int(s.view(torch.uint64).item()),
               int(w.view(torch.uint64).item()), mx))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_are_aligned_and_cover():
    for n in (0, 1, 2047, 2048, N, 1 << 32):
        for world in (1, 2, 4, 8):
            rs = [D.shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, _) in zip(rs, rs[1:]):
                assert b == c and a <= b and a % 2048 == 0
            if n == 1 << 32:
                assert all(b - a == n // world for a, b in rs)


def test_two_rank_gloo_matches_single_column_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-column oracle
    X = O.encode(synth.gen_host("c5.X", N), O.DYN_BP, 0, 512)
    Y = O.encode(synth.gen_host("c5.Y", N), O.FOR_BP, 0, 512)
    pos = O.select(X, O.LT, SEL, out_fmt=O.DELTA_BP, out_block=512)
    expect_pos = O.decode(pos)
    expect_sum = O.agg_sum(O.project(Y, pos, 0, O.FOR_BP, 0, 512))
    counts = res[0][3]
    assert all(r[3] == counts for r in res)
    assert sum(counts) == pos.n
    got = np.concatenate([np.asarray(r[5], dtype=np.uint64) for r in res])
    assert np.array_equal(got, expect_pos)
    for r in res:  # C1 offsets place each shard's positions at their global ranks
        off = r[4][r[0]]
        assert np.array_equal(np.asarray(r[5], dtype=np.uint64), expect_pos[off:off + counts[r[0]]])
    assert all(r[6] == expect_sum for r in res)
    assert all(r[7] == 0 for r in res)
    assert all(r[8] == 2.0 for r in res)
