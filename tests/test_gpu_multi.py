"""BJ.c5's sharded chain under NCCL: one process per
GPU, row-range shards, select with global row ids, C1 allgather of the counts ->
output offsets, project of the co-sharded Y, C2 allreduce of the sums mod 2^64.
Every shard's positions and Y' images must equal the oracle's over the shard's
rows, and the assembled result the single-column oracle's.

World size 1 always runs (it exercises the NCCL code path of the collectives on
one GPU, no rank waits on another); world size 2 runs when two GPUs are visible."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

N = (1 << 22) + 2048 * 5 + 100
SEL = 1 << 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from paper_2004_09350_b200 import dist as D
        from paper_2004_09350_b200 import ms
        start, end = D.shard_range(N, world, rank)
        X = ms.compress(synth.gen_torch("c5.X", end - start, start=start), ms.dyn_bp(512))
        Y = ms.compress(synth.gen_torch("c5.Y", end - start, start=start), ms.for_bp(512))
        pos = ms.select(X, ms.LT, SEL, row_offset=start, out_fmt=ms.delta_bp(512))
        counts = D.allgather_counts(pos.n, dev)
        yp = ms.project(Y, pos, start, ms.for_bp(512))
        s = ms.agg_sum(yp, check=True)
        D.allreduce_u64_sum(s)
        wrap = torch.tensor([-(1 << 63)], dtype=torch.int64, device=dev)  # 2^63 from every rank
        D.allreduce_u64_sum(wrap)
        mx = D.max_over_ranks(float(rank + 1), dev)
        q.put((rank, start, end, counts, pos.images(), yp.images(), ms.u64(s), ms.u64(wrap), mx))
    finally:
        dist.destroy_process_group()


def _run(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _check(res, world):
    counts = res[0][3]
    assert all(r[3] == counts for r in res)
    offs = np.cumsum([0] + counts[:-1]).tolist()
    X = O.encode(synth.gen_host("c5.X", N), O.DYN_BP, 0, 512)
    Y = O.encode(synth.gen_host("c5.Y", N), O.FOR_BP, 0, 512)
    opos = O.select(X, O.LT, SEL, out_fmt=O.DELTA_BP, out_block=512)
    expect_pos = O.decode(opos)
    expect_sum = O.agg_sum(O.project(Y, opos, 0, O.FOR_BP, 0, 512))
    assert sum(counts) == opos.n
    for rank, start, end, _, pimg, yimg, s, wrap, mx in res:
        m = end - start
        sx = O.encode(synth.gen_host("c5.X", m, start), O.DYN_BP, 0, 512)
        sy = O.encode(synth.gen_host("c5.Y", m, start), O.FOR_BP, 0, 512)
        spos = O.select(sx, O.LT, SEL, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
        syp = O.project(sy, spos, start, O.FOR_BP, 0, 512)
        for sec in ("payload", "cw", "ref", "rem"):
            assert np.array_equal(pimg[sec], getattr(spos, sec)), (rank, "positions", sec)
            assert np.array_equal(yimg[sec], getattr(syp, sec)), (rank, "Y'", sec)
        dec = O.decode(spos)  # C1: the shard's positions sit at its global output ranks
        assert np.array_equal(dec, expect_pos[offs[rank]:offs[rank] + counts[rank]])
        assert s == expect_sum
        assert wrap == ((1 << 63) * world) % (1 << 64)
        assert mx == float(world)


def test_nccl_world_size_1():
    _check(_run(1), 1)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs (one process per GPU)")
def test_nccl_world_size_2():
    _check(_run(2), 2)
