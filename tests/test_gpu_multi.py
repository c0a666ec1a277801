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
        gcol, ka, cw_off = D.reblock_positions(pos)  # K11: this rank's slice of the global column
        q.put((rank, start, end, counts, pos.images(), yp.images(), ms.u64(s), ms.u64(wrap), mx,
               (gcol.images(), cw_off)))
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
    glob = _assemble([r[9] for r in res])  # K11: the re-blocked global column
    for sec in ("payload", "cw", "ref", "rem"):
        assert np.array_equal(glob[sec], getattr(opos, sec)), ("K11", sec)
    for rank, start, end, _, pimg, yimg, s, wrap, mx, _g in res:
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


def _assemble(parts):
    """Global image from the ranks' re-blocked slices: payloads and refs in rank
    order, cw shifted by each rank's offset, the remainder from the last rank."""
    pay, cw, ref = [], [np.zeros(1, np.uint32)], []
    for img, off in parts:
        pay.append(img["payload"])
        cw.append((img["cw"][1:].astype(np.uint64) + np.uint64(off)).astype(np.uint32))
        ref.append(img["ref"])
    return {"payload": np.concatenate(pay), "cw": np.concatenate(cw), "ref": np.concatenate(ref),
            "rem": parts[-1][0]["rem"]}


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("sel", [1 << 16, 1 << 9, 3])
def test_k11_global_reblocking_emulated(G, sel):
    """K11: G row-range shards selected on one GPU, then re-blocked
    into ONE global DELTA_BP{512} column (heads from the predecessors' tails, cw
    offsets from the ranks' width totals) — byte-identical to the single-column
    oracle image, including shards that own no full block (sel = 3: a handful of
    matches in the whole column)."""
    from paper_2004_09350_b200 import dist as D
    from paper_2004_09350_b200 import ms
    n = (1 << 21) + 2048 * 7 + 333
    contrib = []
    for s in range(G):
        start, end = D.shard_range(n, G, s)
        X = ms.compress(synth.gen_torch("c5.X", end - start, start=start), ms.dyn_bp(512))
        pos = ms.select(X, ms.LT, sel, row_offset=start, out_fmt=ms.delta_bp(512))
        contrib.append(D.reblock_contribution(pos))
    counts = [c[0] for c in contrib]
    tails = [c[1] for c in contrib]
    parts, wsum = [], 0
    for s in range(G):
        col, ka = D.reblock_local(contrib[s][2], s, counts, tails)
        parts.append((col.images(), wsum))
        wsum += col.payload_words * 64 // 512
    got = _assemble(parts)
    X = O.encode(synth.gen_host("c5.X", n), O.DYN_BP, 0, 512)
    want = O.select(X, O.LT, sel, out_fmt=O.DELTA_BP, out_block=512)
    for sec in ("payload", "cw", "ref", "rem"):
        assert np.array_equal(got[sec], getattr(want, sec)), (G, sel, sec)
