#!/usr/bin/env python3
"""bench.py — the hot path of MorphStore's compression-enabled processing model
on B200, measured on BASELINE.json configs[4] ("c5", the configuration the
metric is quoted on at 1/2/4/8 GPUs; it fits one GPU: 2^32 values).

One step = one pass of the whole hot path over the resident compressed columns:
  select(X DYN_BP{512}, X < 2^16) -> positions DELTA_BP{512} (global row ids)
  [N>1: C1 allgather of the per-shard counts]
  project(Y FOR_BP{512}, positions) -> Y' FOR_BP{512}
  agg_sum(Y') -> uint64
  [N>1: C2 allreduce of the per-shard sums]
Inputs are seeded synthetic columns (synth/), generated on
the device shard by shard and compressed by libms before the timed region.
Inputs (10.8 + 10.9 GB at N=1) are far larger than L2 (126 MB): no L2 flush.

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
(or plain `python bench.py --gpus N`: without WORLD_SIZE in the environment the
script re-launches itself under torch.distributed.run, one rank per GPU, with
NCCL_DEBUG=INFO unless set).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "select+recompress Gvalues/s and HBM GB/s vs ~8 TB/s peak at 1/2/4/8 B200"
UNIT = "Gvalues/s"
N_C5 = 1 << 32
SEL_C5 = 1 << 16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c5"])
    ap.add_argument("--n-log2", type=int, default=32, help="rows of c5 (default 2^32, the config's size)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity-gate", action="store_true", help="(experiments) report instead of exiting on a parity failure")
    ap.add_argument("--pos-fmt", default="delta_bp:512", help="(experiments) positions format, e.g. uncompr")
    ap.add_argument("--proj-fmt", default="for_bp:512", help="(experiments) projected column format")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


NOMINAL_HBM_GBS = 8000.0  # BASELINE.json north_star's "~8 TB/s"


def host_info():
    """The host the CPU legs run on: logical CPUs, model name, and the pinning used."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


class pinned_to_one_core:
    """Pin this process to one CPU for the oracle timing (the paper's single-thread
    setup); restores the previous affinity."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.cpu = min(self.prev)
        os.sched_setaffinity(0, {self.cpu})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.prev)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clock / throttle-reason samples during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.gpu_id)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


# ------------------------------------------------------------ reference arm
def oracle_sample(n_s: int, start: int = 0):
    """Encode a bounded sample of c5 with the oracle (untimed); returns (X, Y) images."""
    import oracle as O
    import synth
    X = O.encode(synth.gen_host("c5.X", n_s, start), O.DYN_BP, 0, 512)
    Y = O.encode(synth.gen_host("c5.Y", n_s, start), O.FOR_BP, 0, 512)
    return X, Y


def oracle_step(X, Y, start=0):
    """The same hot path, by the oracle: select -> project -> sum (decode / encode
    literally, operators on the decoded vectors)."""
    import oracle as O
    pos = O.select(X, O.LT, SEL_C5, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
    yp = O.project(Y, pos, start, O.FOR_BP, 0, 512)
    return O.agg_sum(yp), pos


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    n_s = 1 << 22
    X, Y = oracle_sample(n_s)
    with pinned_to_one_core() as pin:
        for _ in range(args.warmup):
            oracle_step(X, Y)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle_step(X, Y)
        t = time.perf_counter() - t0
    v = n_s * args.steps / t / 1e9
    sample = (f"c5 rows [0, 2^22) per step (X DYN_BP{{512}}, Y FOR_BP{{512}}): select X<2^16 -> DELTA_BP{{512}}, "
              f"project Y -> FOR_BP{{512}}, sum; oracle = plain C, one thread")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (counter-based splitmix64, SURVEY.md §8(d) d.2)",
            "config": {"workload": "c5 (BASELINE.json configs[4]) bounded CPU sample", "rows_per_step": n_s},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "pinned_cpu": pin.cpu, **host_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- our arm
def cpu_baseline_ours():
    """Oracle timed on a bounded sample of the same workload, on this host, one thread."""
    n_s = 1 << 24
    X, Y = oracle_sample(n_s)
    with pinned_to_one_core() as pin:
        t0 = time.perf_counter()
        oracle_step(X, Y)
        t = time.perf_counter() - t0
    return {"value": n_s / t / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "c5 rows [0, 2^24): select X<2^16 -> DELTA_BP{512}, project Y -> FOR_BP{512}, sum "
                      "(plain-C oracle, single thread, inputs pre-encoded)",
            "seconds": t, "pinned_cpu": pin.cpu, **host_info()}


def touched_gather_bytes(X, Y, start, pos_fmt):
    """Algorithmic bytes of the gather: the positions image
    plus the distinct 32-byte sectors of Y's payload the selected codes occupy plus
    the header entries (cw, ref) of the touched blocks. Computed once, outside the
    timed region, with torch on the device (bench accounting only)."""
    import numpy as np
    import torch
    from paper_2004_09350_b200 import ms
    pos = ms.select(X, ms.LT, SEL_C5, row_offset=start, out_fmt=pos_fmt)
    p = ms.decompress(pos) - start
    img = Y.images()
    cw = torch.from_numpy(img["cw"].astype(np.int64)).cuda()
    b = p >> 9
    w = cw[b + 1] - cw[b]
    bit = cw[b] * 512 + (p & 511) * w
    nsec = (Y.payload_words * 64 + 255) // 256
    mark = torch.zeros(nsec + 1, dtype=torch.bool, device="cuda")
    mark[bit >> 8] = True
    mark[(bit + w - 1).clamp(min=0) >> 8] = True
    sectors = int(mark.sum().item())
    blocks = int(torch.unique_consecutive(b).numel())
    out = pos.footprint() + 32 * sectors + blocks * (4 + 8)
    del p, b, w, bit, mark, cw, pos
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as tdist

    import synth
    from paper_2004_09350_b200 import dist as D
    from paper_2004_09350_b200 import ms

    rank, world, local = env_rank()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)
    n = 1 << args.n_log2
    start, end = D.shard_range(n, world, rank)
    m = end - start

    # ---- setup: generate + compress this rank's shard (untimed)
    x = synth.gen_torch("c5.X", m, start=start)
    X = ms.compress(x, ms.dyn_bp(512))
    del x
    y = synth.gen_torch("c5.Y", m, start=start)
    Y = ms.compress(y, ms.for_bp(512))
    del y
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    def parse_fmt(spec):
        name, _, arg = spec.partition(":")
        return getattr(ms, name)(int(arg)) if arg else getattr(ms, name)()

    pos_fmt, proj_fmt = parse_fmt(args.pos_fmt), parse_fmt(args.proj_fmt)

    def step():
        pos = ms.select(X, ms.LT, SEL_C5, row_offset=start, out_fmt=pos_fmt)
        counts = D.allgather_counts(pos.n, dev) if world > 1 else [pos.n]
        yp = ms.project(Y, pos, start, proj_fmt)
        s = ms.agg_sum(yp)
        if world > 1:
            D.allreduce_u64_sum(s)
        return pos, yp, s, counts

    # ---- parity of the measured configuration against the survey anchors
    pos, yp, s, counts = step()
    total_sel = sum(counts)
    gsum = ms.u64(s)
    parity = {"selected": total_sel, "sum": gsum}
    apath = os.path.join(ROOT, "tests", "golden", "config_anchors.json")  # written by tools/make_anchors.py (oracle)
    if args.n_log2 == 32 and os.path.exists(apath):
        a5 = json.load(open(apath))["c5"]
        parity["expected_selected"] = a5["count"]
        parity["expected_sum"] = a5["sum_projected"]
        parity["ok"] = total_sel == a5["count"] and gsum == a5["sum_projected"]
        if not parity["ok"] and not args.no_parity_gate:
            print(json.dumps({"error": "parity failure", "parity": parity}), flush=True)
            return 1
    bytes_pos, bytes_yp = pos.footprint(), yp.footprint()
    del pos, yp, s

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()

    props = torch.cuda.get_device_properties(local)
    sampler = ClockSampler(f"GPU-{props.uuid}" if hasattr(props, "uuid") else local)
    if rank == 0:
        sampler.start()
    ms.profile_read()
    ms.profile_enable(True)
    l0 = ms.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    launches = ms.launch_count() - l0
    ms.profile_enable(False)
    prof = ms.profile_read()
    ms_total = e0.elapsed_time(e1)
    if world > 1:
        ms_total = D.max_over_ranks(ms_total, dev)
        tdist.barrier()
    clocks = sampler.stop() if rank == 0 else None

    # ---- roofline of the dominant kernel (algorithmic bytes / event-timed duration)
    peak, peak_src = peaks()
    x_bytes, y_bytes = X.footprint(), Y.footprint()
    gather_bytes = touched_gather_bytes(X, Y, start, pos_fmt)  # positions + touched Y sectors/headers
    # algorithmic bytes per launch: what the method itself must move
    mask_bytes = 4 * 16 * ((m + 511) // 512)                       # select's 1-bit-per-row match mask
    alg = {"select_fast": x_bytes + mask_bytes,                    # compressed X read, mask written
           "select_stream": x_bytes + mask_bytes,
           "pos_width": mask_bytes,                                # mask read
           "pos_pack": mask_bytes + bytes_pos,                     # mask read, positions image written
           "pos_encode": mask_bytes + bytes_pos,
           "pos_slot": mask_bytes + bytes_pos,                     # mask read, blocks written to slots
           "pos_copy": 2 * bytes_pos,                              # slots read, positions image written
           "project_fast": gather_bytes + bytes_yp,                # positions + touched Y + Y' written
           "project_pipe": gather_bytes + bytes_yp,
           "project_win": gather_bytes + bytes_yp,
           "project_slot": gather_bytes + bytes_yp,                # positions + touched Y + Y' into slots
           "project_stream": gather_bytes + bytes_yp,              # positions + touched Y + Y' into slots
           "project_copy": 2 * bytes_yp,                           # slots read, Y' written
           "project_warp": gather_bytes + bytes_yp,
           "sum_fast": bytes_yp,                                   # Y' read
           "sum_stream": bytes_yp}
    kernels = {}
    for k, (k_launches, tot_ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        avg = tot_ms / max(1, k_launches)
        ent = {"launches": k_launches, "avg_ms": avg, "share": tot_ms / ms_total}
        if k in alg:
            ent["alg_bytes"] = alg[k]
            ent["achieved_gbs"] = alg[k] / (avg * 1e-3) / 1e9
            ent["frac_of_peak"] = ent["achieved_gbs"] / peak
        kernels[k] = ent
    # ALU roofline of the issue-bound encoder: executed warp instructions per launch
    # (ncu, this build, this workload) over its event-timed duration, against the
    # issue peak (4 schedulers x SMs x the SM clock sampled during the run)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
    clk_mhz = (clocks or {}).get("sm_mhz") or 1965.0
    issue_peak = 4 * props.multi_processor_count * clk_mhz * 1e6
    for k, ins in tj.get("_inst", {}).items():
        if k in kernels and args.n_log2 == 32 and world == 1:
            a = ins / (kernels[k]["avg_ms"] * 1e-3)
            kernels[k]["alu"] = {"warp_inst_per_launch": ins, "achieved_ginst_s": a / 1e9,
                                 "issue_peak_ginst_s": issue_peak / 1e9, "frac": a / issue_peak}
    dom_name = max(prof.items(), key=lambda kv: kv[1][1])[0]
    dom = kernels[dom_name]
    traffic, traffic_src = None, None
    if tj and args.n_log2 == 32 and world == 1:  # captured at this workload (one GPU, 2^32 rows)
        traffic = tj.get(dom_name)
        traffic_src = tj.get("_about")
    step_ms = ms_total / args.steps
    chain_alg = x_bytes + bytes_pos + gather_bytes + 2 * bytes_yp
    value = n * args.steps / (ms_total * 1e-3) / 1e9

    # ---- e2e: host images -> device -> chain -> 8-byte result back, every step
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, X, Y, start, world, dev, n)
    del X, Y
    torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline_ours()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (counter-based splitmix64, SURVEY.md §8(d) d.2)",
            "config": {"workload": "c5 (BASELINE.json configs[4]): select X<2^16 -> DELTA_BP{512} -> project Y "
                                   "-> FOR_BP{512} -> sum", "rows": n, "X": "DYN_BP{512}", "Y": "FOR_BP{512}",
                       "parallelism": f"row-range shards x{world}", "l2_flush": "none: inputs >> 126 MB L2",
                       "X_bytes": x_bytes * (world if world > 1 else 1), "Y_bytes": y_bytes},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": dom.get("achieved_gbs"), "peak": peak,
                         "unit": "GB/s", "frac": dom.get("frac_of_peak"), "traffic": traffic,
                         "frac_nominal": (dom.get("achieved_gbs") or 0) / NOMINAL_HBM_GBS,
                         "nominal_peak": NOMINAL_HBM_GBS,
                         "alg_bytes_per_launch": dom.get("alg_bytes"), "avg_launch_ms": dom["avg_ms"],
                         "peak_source": peak_src, "traffic_source": traffic_src},
            "hbm_gbs_chain": chain_alg / (step_ms * 1e-3) / 1e9,
            "chain_frac": chain_alg / (step_ms * 1e-3) / 1e9 / peak,
            "chain_frac_nominal": chain_alg / (step_ms * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
            "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


def run_e2e(args, X, Y, start, world, dev, n):
    """The same chain through the C ABI with HOST buffers: each step uploads the
    compressed X and Y images from pinned host memory (ms_column_to_device),
    runs select -> project -> sum and reads the 8-byte result back."""
    import torch
    from paper_2004_09350_b200 import dist as D
    from paper_2004_09350_b200 import ms
    import ctypes

    def pinned_images(col):
        img = col.images()
        out = {}
        for k, a in img.items():
            t = torch.empty(a.size, dtype=torch.int64 if a.dtype == "uint64" else torch.int32, pin_memory=True)
            if a.size:
                t.numpy().view(a.dtype)[:] = a
            out[k] = t
        return out

    hx, hy = pinned_images(X), pinned_images(Y)

    def host_desc(col, imgs):
        h = ms._Column()
        h.fmt = col._c.fmt
        h.n, h.n_blocks, h.n_rem, h.n_runs = col._c.n, col._c.n_blocks, col._c.n_rem, col._c.n_runs
        h.payload_words = col._c.payload_words
        for k in ("payload", "cw", "ref", "rem"):
            setattr(h, k, imgs[k].data_ptr() if imgs[k].numel() else None)
        return h

    dx, dy = host_desc(X, hx), host_desc(Y, hy)
    h2d = X.footprint() + Y.footprint()
    res = torch.empty(1, dtype=torch.int64, pin_memory=True)
    stream = torch.cuda.current_stream()

    def step():
        cx, cy = ms._Column(), ms._Column()
        ms._check(ms.lib().ms_column_to_device(ctypes.byref(ms._ctx()), ctypes.byref(dx), ctypes.byref(cx)), "h2d")
        ms._check(ms.lib().ms_column_to_device(ctypes.byref(ms._ctx()), ctypes.byref(dy), ctypes.byref(cy)), "h2d")
        Xd, Yd = ms.Column(cx), ms.Column(cy)
        pos = ms.select(Xd, ms.LT, SEL_C5, row_offset=start, out_fmt=ms.delta_bp(512))
        if world > 1:
            D.allgather_counts(pos.n, dev)
        yp = ms.project(Yd, pos, start, ms.for_bp(512))
        s = ms.agg_sum(yp)
        if world > 1:
            D.allreduce_u64_sum(s)
        res.copy_(s, non_blocking=True)
        stream.synchronize()
        return int(res.item())

    k = max(1, min(args.steps, 3))
    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    if world > 1:
        t = D.max_over_ranks(t, dev)
    return {"value": n * k / t / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d * (world if world > 1 else 1),
            "d2h_bytes_per_step": 8, "steps": k, "ms_per_step": 1e3 * t / k,
            "note": "pinned host images -> ms_column_to_device -> select -> project -> sum -> 8 B result"}


def self_launch(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: re-run this script under
    torch.distributed.run, one rank per GPU; rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
