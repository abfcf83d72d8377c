#!/usr/bin/env python3
"""Benchmark of the B200 shape-adaptive motion-estimation hot path.

Default workload (BASELINE.json config 4, the throughput batch): 256
independent CIF 352x288 sequences x 30 frames from the config-2 generator
(seed = base + i), proposed algorithm (PA: BRS + PRS) at +/-16, 8x8 blocks,
ref_distance 2, with motion compensation + PSNR (SSE) of every pair.  One
"step" = one pass of the whole pipeline (classify -> wavefront sort -> PA
search with the fused SSE) over the batch.  Metric: macroblocks/s =
(W/16)(H/16) x pairs x sequences / s, every 16x16 macroblock counted
(transparent ones included).

The same run also measures BASELINE's second headline, exhaustive search on
config 5 (4K, 30 frames = 28 pairs, S = 64, 16x16) on the INT pipe: the
`es_cfg5` object of the JSON line (its own clocks, roofline against the
VABSDIFF4 peak measured live, a reference CPU sample, sampled parity).

  python bench.py [--gpus N --steps K --warmup W] [--workload cfg4-pa|cfg5-es|...]
  python bench.py --impl reference ...   # the reference's own CPU code path

Multi-GPU (one process per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run): config 4 is STRONG-scaled by default — the 256
sequences are sharded over the ranks (`--weak`: 256 per rank) — and each
step's MV fields + per-pair stats/SSE are gathered into rank 0 over NCCL,
overlapped with the next step.  ES config 5 shards (pair, block-row band)
units over the ranks, balanced by estimated-block count.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# workload -> (config id, algo, block size, search range, default sequences)
WORKLOADS = {
    "cfg4-pa": (4, "PA", 8, 16, 256),
    "cfg2-pa": (2, "PA", 8, 16, 1),
    "cfg2-es": (2, "ES", 16, 16, 1),
    "cfg1-pa": (1, "PA", 8, 16, 1),
    "cfg3-pa": (3, "PA", 8, 32, 1),
    "cfg3-tss": (3, "TSS", 16, 32, 1),
    "cfg3-fss": (3, "FSS", 16, 32, 1),
    "cfg3-ds": (3, "DS", 16, 32, 1),
    "cfg5-es": (5, "ES", 16, 64, 1),
    "cfg5-pa": (5, "PA", 8, 64, 1),
    "cfg5-tss": (5, "TSS", 16, 64, 1),
    "cfg5-fss": (5, "FSS", 16, 64, 1),
    "cfg5-ds": (5, "DS", 16, 64, 1),
}
ALGO_ID = {"ES": 0, "TSS": 1, "FSS": 2, "DS": 3, "PA": 4}
BASE_SEED = 20260000
GEOMETRY = {1: "QCIF 176x144", 2: "CIF 352x288", 3: "1920x1088", 4: "CIF 352x288", 5: "3840x2160"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every
    `interval` seconds by a background thread DURING the timed region."""

    SLOW = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown", "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
            "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown", "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
            "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, device_index, interval=0.001):
        self.device, self.interval = device_index, interval
        self.samples, self.thread, self.err = [], None, None

    def _handle(self, nv):
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            return nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.device)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv, self.h = nv, self._handle(nv)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: the line says so
            self.err = f"nvml unavailable: {e}"
            return self
        self.stop_flag = False

        def run():
            nv, h = self.nv, self.h
            bits = {k: getattr(nv, v, 0) for k, v in self.SLOW.items()}
            while not self.stop_flag:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, [k for k, b in bits.items() if b and (r & b)]))
                except Exception as e:
                    self.err = str(e)
                    return
                time.sleep(self.interval)

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()
        return self

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"], "samples": 0, "source": "nvml"}
        self.stop_flag = True
        self.thread.join(timeout=2)
        sm = [s for s, _ in self.samples]
        reasons = sorted({r for _, rs in self.samples for r in rs})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.max_mhz), "reasons": reasons,
                "samples": len(sm), "source": f"NVML every {self.interval * 1e3:.0f} ms during the timed region"}


def respawn_torchrun(args_list, n):
    """`--gpus N` without a torchrun environment: re-launch this script as N
    ranks (one process per GPU) and return their exit code."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + args_list
    log("[bench] launching", " ".join(cmd))
    return subprocess.call(cmd)


def me_config(algo, bs, S):
    import paper_1002_1168_b200 as me

    return me.BatchConfig(algo=me.Algo[algo], search=me.SearchConfig(search_range=S, block_size=bs, ref_distance=2), prs=me.PrsConfig())


def workload_config(wl, args, world, n_total, F):
    cfg_id, algo, bs, S, _ = WORKLOADS[wl]
    strong = cfg_id == 4 and not args.weak
    c = {
        "workload": f"{wl}: BASELINE config {cfg_id} ({GEOMETRY[cfg_id]} x {F}f, {F - 2} pairs), {algo} S={S} bs={bs}, ref_distance 2"
        + (f", {n_total} sequences in total ({'sharded over' if strong else 'per rank,'} {world} GPU(s))" if cfg_id == 4 else ""),
        "config_id": cfg_id,
        "algo": algo,
        "search_range": S,
        "block_size": bs,
        "frames": F,
        "sequences": n_total,
        "l2": "inputs larger than L2 (126 MB)" if cfg_id in (3, 4, 5) else "L2 flushed between steps (256 MB write)",
        "parallelism": (f"dp{world}: sequences sharded (strong), per-step gather of MV fields + pair stats/SSE to rank 0 over NCCL, overlapped with the next step"
                        if strong else f"dp{world}: {'independent batches per rank (weak)' if cfg_id == 4 else 'replicas'}"),
    }
    return c


# ---------------------------------------------------------------------------
# Reference arm: the reference's own CPU code path (oracle/_ref/libme_ref.so,
# the unmodified reference sources), inputs from the same generator compiled
# into that library (oracle/ref_synth_glue.cpp) — libme_b200.so is never loaded.


def cpu_sample(wl, luma, alpha, threads, kind_pref="reference"):
    """Times the reference on a bounded sample of the workload with `threads`
    host threads.  Returns (MB/s, sample text, seconds, kind)."""
    import oracle as O

    cfg_id, algo, bs, S, _ = WORKLOADS[wl]
    kind = "reference" if O.available("reference") else "port"
    orc = O.Oracle(kind)
    cfg = O.make_cfg(algo=ALGO_ID[algo], search_range=S, block_size=bs, ref_distance=2)
    n_seq, F, H, W = luma.shape
    mbpp = (W // 16) * (H // 16)
    if algo == "PA":  # one sequence per thread (pairs chain through the temporal candidate)
        t = time.perf_counter()
        orc.time_sequences(cfg, np.ascontiguousarray(luma), np.ascontiguousarray(alpha), threads)
        dt = time.perf_counter() - t
        return n_seq * (F - 2) * mbpp / dt, f"{n_seq} sequences x {F - 2} pairs ({kind}, {threads} threads)", dt, kind
    if algo in ("TSS", "FSS", "DS"):
        n_pairs = F - 2
        t = time.perf_counter()
        orc.time_pairs(cfg, luma[0], alpha[0], 0, n_pairs, threads)
        dt = time.perf_counter() - t
        return n_pairs * mbpp / dt, f"1 sequence x {n_pairs} pairs ({kind}, {threads} threads)", dt, kind
    # ES: a bounded sample of pair 0's estimated blocks, scaled to whole pairs
    types = orc.classify(alpha[0, 2], bs)
    cols = W // bs
    est = np.flatnonzero(types != 0)
    k = min(est.size, max(threads * 4, 16))
    pick = est[np.linspace(0, est.size - 1, k).astype(int)]
    xy = np.stack([(pick % cols) * bs, (pick // cols) * bs], 1).astype(np.int32)
    t = time.perf_counter()
    orc.time_blocks(cfg, np.ascontiguousarray(luma[0, 2]), np.ascontiguousarray(luma[0, 0]), xy, threads)
    dt = time.perf_counter() - t
    return k / dt * mbpp / est.size, f"{k} of {est.size} estimated blocks of pair 0 ({kind}, {threads} threads), scaled to whole pairs", dt, kind


def ref_inputs(cfg_id, n, first_seed, F, threads):
    import oracle as O

    return O.synth_batch(cfg_id, n, first_seed, F, threads=threads)


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg_id, algo, bs, S, nseq = WORKLOADS[wl]
    threads = os.cpu_count() or 1
    F = args.frames or {1: 10, 2: 30, 3: 60, 4: 30, 5: 30}[cfg_id]
    n_total = (args.n_seq or nseq) if cfg_id == 4 else 1
    # bounded sample: up to 4 sequences per host thread (a few CPU-seconds)
    n = min(n_total, max(16, 4 * threads)) if cfg_id == 4 else 1
    luma, alpha = ref_inputs(cfg_id, n, BASE_SEED, F, threads)
    vals, sample, kind = [], "", "reference"
    for i in range(args.warmup + args.steps):
        v, sample, dt, kind = cpu_sample(wl, luma, alpha, threads)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    one = one_core(wl, luma, alpha)
    gpus = int(os.environ.get("WORLD_SIZE", args.gpus))
    line = {
        "impl": "reference",
        "metric": "macroblocks/sec",
        "value": value,
        "unit": "MB/s",
        "n_gpus": gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "strong" if cfg_id == 4 and not args.weak else "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (seeded integer config generator, SURVEY §8d), generated by oracle/_ref (no libme_b200.so in this arm)",
        "config": workload_config(wl, args, gpus, n_total, F),
        "cpu_baseline": {"value": value, "unit": "MB/s", "cores": threads, "kind": kind, "sample": sample, **one},
        "e2e": {"value": value, "unit": "MB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def one_core(wl, luma, alpha):
    """The same reference code on ONE host thread over a small sample."""
    cfg_id = WORKLOADS[wl][0]
    n1 = min(luma.shape[0], 4) if cfg_id == 4 else 1
    v1, s1, dt1, _ = cpu_sample(wl, luma[:n1], alpha[:n1], 1)
    return {"value_1core": v1, "seconds_1core": dt1, "sample_1core": s1}


# ---------------------------------------------------------------------------
# b200 arm


def digest_parity(recs_np, stats_np, luma_h, alpha_h, cfg_id, algo, bs, S, threads):
    """Checks the CUDA path's MV fields + stats of a batch against the
    reference's own results on the same inputs (per-sequence digests,
    oracle/ref_driver.cpp Digest).  Returns (parity dict, reference seconds)."""
    import oracle as O

    n_seq, F, H, W = luma_h.shape
    cfg = O.make_cfg(algo=ALGO_ID[algo], search_range=S, block_size=bs, ref_distance=2)
    t = time.perf_counter()
    want = O.time_sequences_digest(cfg, luma_h, alpha_h, threads)
    dt = time.perf_counter() - t
    got = O.digest_records(recs_np, stats_np, W, H)
    bad = np.flatnonzero(got != want)
    return {"sequences": int(n_seq), "mismatches": int(bad.size), "first_bad": [int(i) for i in bad[:8]],
            "how": "per-sequence digest of every MV, the SearchStats counters and the exact SSE vs the reference (oracle/_ref) on the same inputs"}, dt


def bench_pa_batch(args, wl, world, rank, local, dev):
    """Config 4 (or any PA/baseline batch workload): returns the JSON line (rank 0) or None."""
    import torch
    import torch.distributed as dist

    import paper_1002_1168_b200 as me
    from paper_1002_1168_b200 import _lib
    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import dist as mdist
    from paper_1002_1168_b200 import synth

    cfg_id, algo, bs, S, nseq_default = WORKLOADS[wl]
    n_arg = args.n_seq or nseq_default
    strong = cfg_id == 4 and not args.weak
    if cfg_id == 4:
        if strong:
            counts = [mdist.shard(n_arg, r, world)[1] for r in range(world)]
            first = mdist.shard(n_arg, rank, world)[0]
            n_total = n_arg
        else:
            counts = [n_arg] * world
            first = rank * n_arg
            n_total = n_arg * world
    else:
        counts, first, n_total = [1] * world, 0, world
    n_seq = counts[rank]
    F = args.frames or {1: 10, 2: 30, 3: 60, 4: 30, 5: 30}[cfg_id]
    warmup = max(args.warmup, 3)
    t0 = time.perf_counter()
    luma, alpha = synth.config4_batch_dev(n_seq, BASE_SEED + first, F, config_id=cfg_id, device=local)
    torch.cuda.synchronize(dev)
    H, W = luma.shape[2], luma.shape[3]
    log(f"[rank {rank}] generated {n_seq} x {F} x {H}x{W} on the device in {time.perf_counter() - t0:.2f}s")
    cfg = me_config(algo, bs, S)
    pairs = F - 2
    rows, cols = H // bs, W // bs
    recs = torch.empty((n_seq, pairs, rows, cols, 16), dtype=torch.uint8, device=dev)
    stats = torch.empty((n_seq, pairs, 48), dtype=torch.uint8, device=dev)
    gatherer = mdist.ResultGatherer(S, counts) if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if cfg_id in (1, 2) else None
    stream = torch.cuda.current_stream(dev)
    lib = me.lib()
    ctxh = _lib.ctx(local)
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))
    import ctypes as C

    stage = (C.c_float * 4)()
    stage_sum = np.zeros(4)

    def step(stages):
        B.run_sequences_dev(cfg, luma, alpha, recs, stats, device=local, stream=stream.cuda_stream)
        if stages:  # waits for the step: only in the untimed breakdown pass below
            _lib.check(lib.me_b200_ctx_stage_ms(ctxh, stage, 4))
            stage_sum[:] += np.array(stage[:])
        if gatherer is not None:  # step k's MV fields + stats -> rank 0, overlapping step k+1
            gatherer.submit(recs, stats)
        if flush is not None:
            flush.fill_(1)

    for _ in range(warmup):
        step(False)
    if gatherer is not None:
        gatherer.finish()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local).start()
    if flush is None:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step(False)
        gathered = gatherer.finish() if gatherer is not None else None  # the last gather completes inside the timed region
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        ms_dev = ev0.elapsed_time(ev1)
    else:  # small single sequences: every step timed by its own events, the L2 flush between them untimed
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for ea, eb in evs:
            ea.record(stream)
            B.run_sequences_dev(cfg, luma, alpha, recs, stats, device=local, stream=stream.cuda_stream)
            eb.record(stream)
            if gatherer is not None:
                gatherer.submit(recs, stats)
            flush.fill_(1)
        gathered = gatherer.finish() if gatherer is not None else None
        torch.cuda.synchronize(dev)
        ms_dev = sum(ea.elapsed_time(eb) for ea, eb in evs)
    clk = clocks.stop()
    launches_per_step = B.last_launches(local)
    ms = mdist.max_over_ranks(ms_dev, dev)
    ms_per_step = ms / args.steps
    total_units = n_total * pairs * (W // 16) * (H // 16)
    value = total_units / (ms_per_step / 1e3)
    compute_only = None
    if gatherer is not None:  # compute-only beside compute + gather (the line's value)
        dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats, device=local, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        c_ms = mdist.max_over_ranks(e0.elapsed_time(e1), dev) / args.steps
        compute_only = {"ms_per_step": c_ms, "value": total_units / (c_ms / 1e3), "unit": "MB/s",
                        "note": "the same steps without the per-step gather to rank 0 (max over ranks)"}
    # per-stage breakdown (CUDA events on the launching stream), untimed
    n_stage = min(args.steps, 20)
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 1))
    for _ in range(n_stage):
        step(True)
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))
    if gatherer is not None:
        gatherer.finish()
    stage_ms = stage_sum / n_stage
    if world > 1:
        dist.barrier()

    # the same batch with the masks resident bit-packed (binary masks: exact;
    # 1/8 of the mask bytes): classify and the PA kernels read the bit planes
    bits_layout = None
    if algo == "PA" and not args.no_bits:
        bits, binary = B.pack_mask_dev(alpha, device=local)
        if world > 1:  # every rank takes the same branch (collectives inside)
            flag = torch.tensor([1 if binary else 0], device=mdist.coll_device(dev))
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            binary = bool(flag.item())
        if binary:
            recs_b = torch.empty_like(recs)
            stats_b = torch.empty_like(stats)
            for _ in range(warmup):
                B.run_sequences_bits_dev(cfg, luma, bits, recs_b, stats_b, device=local, stream=stream.cuda_stream)
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            clocks_b = ClockSampler(local).start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                B.run_sequences_bits_dev(cfg, luma, bits, recs_b, stats_b, device=local, stream=stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            clk_b = clocks_b.stop()
            ms_b = mdist.max_over_ranks(e0.elapsed_time(e1), dev) / args.steps
            _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 1))
            st_b = np.zeros(4)
            for _ in range(n_stage):
                B.run_sequences_bits_dev(cfg, luma, bits, recs_b, stats_b, device=local, stream=stream.cuda_stream)
                _lib.check(lib.me_b200_ctx_stage_ms(ctxh, stage, 4))
                st_b += np.array(stage[:])
            _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))
            st_b /= n_stage
            same = bool(torch.equal(recs_b, recs) and torch.equal(stats_b, stats))
            bytes_b = n_seq * F * W * H * 9 // 8 + n_seq * pairs * rows * cols * 16
            ach_b = bytes_b / (float(st_b.sum()) / 1e3) / 1e9
            bits_layout = {"ms_per_step": ms_b, "value": total_units / (ms_b / 1e3), "unit": "MB/s",
                           "stages_ms": {"classify": st_b[0], "sort": st_b[1], "search": st_b[2], "mc_psnr": st_b[3]},
                           "identical_to_byte_masks": same, "clocks": clk_b,
                           "roofline": {"bound": "hbm", "achieved": ach_b, "peak": peaks()[0], "unit": "GB/s", "frac": ach_b / peaks()[0],
                                        "algorithmic_bytes_per_step": bytes_b},
                           "note": "masks resident in HBM as bit planes (me_b200_run_sequences_bits_dev; packed once by me_b200_pack_mask_dev outside the timed region): 1/8 of the mask bytes, shape SADs as popc(XOR) of bit rows"}
            if not same:
                raise SystemExit("bit-packed mask run differs from the byte-mask run")
            del recs_b, stats_b
        del bits

    # results of the whole batch on rank 0 (the gather's payload at N > 1)
    if world > 1:
        if rank == 0:
            mv_all, st_all = gathered
            recs_np = np.zeros((n_total, pairs, rows, cols), _lib.rec_dtype())
            mv_np = mv_all.cpu().numpy()
            recs_np["dx"], recs_np["dy"] = mv_np[..., 0], mv_np[..., 1]
            stats_np = st_all.cpu().numpy().view(_lib.stats_dtype()).reshape(n_total, pairs)
    else:
        recs_np = recs.cpu().numpy().view(_lib.rec_dtype()).reshape(n_seq, pairs, rows, cols)
        stats_np = stats.cpu().numpy().view(_lib.stats_dtype()).reshape(n_seq, pairs)

    hbm_peak, peak_src = peaks()
    alg_bytes = n_seq * F * W * H * 2 + n_seq * pairs * rows * cols * 16
    pipe_ms = float(stage_ms.sum())
    roof = None
    if algo == "PA":
        traffic, traffic_src = None, None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f).get(wl)
            if tr and tr.get("n_seq") == n_seq:
                traffic, traffic_src = float(sum(tr["dram_bytes"].values())), tr
        ach = alg_bytes / (pipe_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": f"pipeline classify+scan+fill+PA wavefront search ({launches_per_step} launches/step; this rank's shard)",
                "achieved": ach, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic,
                "traffic_by_kernel": traffic_src["dram_bytes"] if traffic_src else None, "algorithmic_bytes_per_step": alg_bytes,
                "pipeline_ms": pipe_ms, "timing": "stage times from CUDA events on the launching stream in an untimed pass right after the timed loop",
                "dominant": {"kernel": "pa_fast + pa_quad + pa_fast (wavefront search)", "ms": float(stage_ms[2]), "share": float(stage_ms[2]) / pipe_ms,
                             "bound": "dependency latency + issue (see DESIGN.md)"}}
    elif rank == 0:  # ES / TSS / FSS / DS: SAD byte-ops (the oracle-exact comparison count x bs^2) on the INT pipe
        ipk = C.c_double()
        _lib.check(lib.me_b200_probe_int_peak(ctxh, C.byref(ipk)))
        ops = float(stats_np["block_comparisons"].sum()) * bs * bs
        ach = ops / (float(stage_ms[2]) / 1e3) / 1e12
        roof = {"bound": "int", "kernel": f"{'es_kernel' if algo == 'ES' else 'ring_kernel'} (search stage)", "achieved": ach,
                "peak": ipk.value / 1e12, "unit": "T byte-ops/s", "frac": ach / (ipk.value / 1e12),
                "peak_source": "VABSDIFF4.U8.ACC microbenchmark measured in this run on this GPU (me_b200_probe_int_peak)",
                "sad_byte_ops_per_step": ops, "search_ms": float(stage_ms[2]),
                "note": "achieved = oracle-exact comparisons x bs^2 byte-ops / search-stage time (CUDA events)"}

    # end to end through the public host-pointer C ABI: pinned H2D + pipeline + D2H
    e2e = None
    hl = ha = None
    need_host = (not args.no_e2e) or (world == 1 and rank == 0)
    if need_host:
        pin = torch.empty((2, n_seq, F, H, W), dtype=torch.uint8, pin_memory=True)
        pin[0].copy_(luma)
        pin[1].copy_(alpha)
        hl, ha = pin[0].numpy(), pin[1].numpy()
    if not args.no_e2e:
        # torchrun sets OMP_NUM_THREADS=1: give each rank its share of the host
        # cores for the mask packing of the host-buffer path
        lws = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        if lws > 1:
            _lib.set_tuning(local, host_threads=max(1, (os.cpu_count() or 1) // lws))
        hrecs = torch.empty((n_seq, pairs, rows, cols, 16), dtype=torch.uint8, pin_memory=True)
        hstats = torch.empty((n_seq, pairs, 48), dtype=torch.uint8, pin_memory=True)
        n_e2e = args.e2e_steps or max(1, min(args.steps, 10))
        B.run_sequences_ptr(cfg, n_seq, F, W, H, hl.ctypes.data, ha.ctypes.data, hrecs.data_ptr(), hstats.data_ptr(), local)  # warm
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(n_e2e):
            B.run_sequences_ptr(cfg, n_seq, F, W, H, hl.ctypes.data, ha.ctypes.data, hrecs.data_ptr(), hstats.data_ptr(), local)
        e2e_s = mdist.max_over_ranks((time.perf_counter() - t) / n_e2e, dev)
        got = hrecs.numpy().view(_lib.rec_dtype()).reshape(n_seq, pairs, rows, cols)
        if not np.array_equal(got, recs.cpu().numpy().view(_lib.rec_dtype()).reshape(n_seq, pairs, rows, cols)):
            raise SystemExit("e2e records differ from the device-resident run")
        h2d, d2h = B.last_transfer_bytes(local)
        probe_h = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        probe_d = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        probe_d.copy_(probe_h, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            probe_d.copy_(probe_h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_gbs = 4 * (256 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9
        del probe_h, probe_d
        e2e = {"value": total_units / e2e_s, "unit": "MB/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": n_e2e,
               "s_per_step": e2e_s, "input_bytes_per_step": int(2 * n_seq * F * W * H), "h2d_gbs_measured": h2d_gbs, "h2d_floor_ms": h2d / h2d_gbs / 1e6,
               "note": "pinned host buffers through me_b200_run_sequences (per rank: its shard); luma as bytes, binary alpha bit-packed on the host cores with all-zero 64-pixel words elided, expanded on the GPU"}

    line = None
    if rank == 0:
        threads = os.cpu_count() or 1
        # the whole batch's inputs on this host: the device-generated bytes at
        # N = 1, the same generator on the host cores otherwise
        if world == 1:
            lh, ah = hl, ha
        else:
            import oracle

            lh, ah = oracle.synth_batch(cfg_id, n_total, BASE_SEED, F, threads=threads) if cfg_id == 4 else oracle.synth_batch(cfg_id, 1, BASE_SEED, F, threads=1)
        parity, ref_s = None, None
        # (replicas of a single-sequence workload at N > 1: rank 0's own result is the check)
        if world > 1 and cfg_id != 4:
            recs_np, stats_np = recs_np[:1], stats_np[:1]
        # (exhaustive search at 4K on the host cores takes minutes: the es_cfg5 leg samples it instead)
        if not args.no_parity and not (algo == "ES" and cfg_id == 5):
            parity, ref_s = digest_parity(recs_np, stats_np, lh, ah, cfg_id, algo, bs, S, threads)
            log(f"[bench] parity vs reference: {parity['mismatches']} of {parity['sequences']} sequences differ")
        cpu = None
        if world == 1 and not args.no_cpu:
            if ref_s is not None:  # the parity run IS the reference on the whole batch, all host threads
                import oracle

                cpu = {"value": n_total * pairs * (W // 16) * (H // 16) / ref_s, "unit": "MB/s", "cores": threads,
                       "kind": "reference" if oracle.available("reference") else "port",
                       "sample": f"the whole batch: {n_total} sequences x {pairs} pairs, {threads} threads (the parity run)", "seconds": ref_s}
            else:
                v, sample, dt, kind = cpu_sample(wl, lh, ah, threads)
                cpu = {"value": v, "unit": "MB/s", "cores": threads, "kind": kind, "sample": sample, "seconds": dt}
            cpu.update(one_core(wl, lh, ah))
        est = int(stats_np["blocks_opaque"].sum() + stats_np["blocks_boundary"].sum())
        line = {
            "metric": "macroblocks/sec",
            "value": value,
            "unit": "MB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic (seeded integer config generator, SURVEY §8d; no public sequences in this container)",
            "config": workload_config(wl, args, world, n_total, F),
            "roofline": roof,
            "stages_ms": {"classify": stage_ms[0], "sort": stage_ms[1], "search": stage_ms[2], "mc_psnr": stage_ms[3]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "parity": parity,
            "bits_layout": bits_layout,
            "estimated_blocks": est,
            "estimated_blocks_per_s": est / (ms_per_step / 1e3),
            "compute_only": compute_only,
            "macroblocks_per_step": int(total_units),
        }
        if parity is not None and parity["mismatches"]:
            print(json.dumps(line), flush=True)
            raise SystemExit(f"parity FAILED: {parity['mismatches']} sequences differ from the reference")
    del luma, alpha, recs, stats
    torch.cuda.empty_cache()
    return line


# ---------------------------------------------------------------------------
# ES on config 5 (the INT-pipe headline), sharded by (pair, row band) units


def bench_critical_path(args, local, dev):
    """PA on the single-sequence configs 1, 2, 3 and 5 (BASELINE.md section 3:
    critical-path bound, not HBM): per configuration the wavefront length
    (steps t = h + 2v + p) and the measured time per step of the search."""
    import torch

    from paper_1002_1168_b200 import _lib
    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import synth
    import ctypes as C

    import paper_1002_1168_b200 as me

    lib, ctxh = me.lib(), _lib.ctx(local)
    stage = (C.c_float * 4)()
    out = {}
    for cid, S in ((1, 16), (2, 16), (3, 32), (5, 64)):
        F = {1: 10, 2: 30, 3: 60, 5: 30}[cid]
        luma, alpha = synth.config4_batch_dev(1, BASE_SEED, F, config_id=cid, device=local)
        cfg = me_config("PA", 8, S)
        H, W = luma.shape[2], luma.shape[3]
        cols, rows, pairs = W // 8, H // 8, F - 2
        steps = (cols - 1) + 2 * (rows - 1) + (pairs - 1) + 1
        recs = torch.empty((1, pairs, rows, cols, 16), dtype=torch.uint8, device=dev)
        stats = torch.empty((1, pairs, 48), dtype=torch.uint8, device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for _ in range(3):
            B.run_sequences_dev(cfg, luma, alpha, recs, stats, device=local)
        _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 1))
        tot, search, n = 0.0, 0.0, 10
        for _ in range(n):
            flush.fill_(1)  # L2 flushed between runs
            B.run_sequences_dev(cfg, luma, alpha, recs, stats, device=local)
            _lib.check(lib.me_b200_ctx_stage_ms(ctxh, stage, 4))
            tot += sum(stage[:4])
            search += stage[2]
        _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))
        tot, search = tot / n, search / n
        est = int(((recs[..., 13] != 0)).sum().item())  # type byte: opaque / boundary
        out[f"cfg{cid}"] = {"geometry": f"{W}x{H} x {F}f, S={S}, 8x8 blocks", "wavefront_steps": steps, "estimated_blocks": est,
                            "pipeline_ms": tot, "search_ms": search, "us_per_step": 1e3 * search / steps,
                            "macroblocks_per_s": pairs * (W // 16) * (H // 16) / (tot / 1e3)}
        del luma, alpha, recs, stats, flush
    torch.cuda.empty_cache()
    return {"model": "search time = wavefront steps x per-step latency (pa_fast_kernel: one CTA per SM with the staged window, S <= 32; two with per-candidate patches, S = 64; CUDA events, L2 flushed)", **out}


def bench_units(args, world, rank, local, dev, wl="cfg5-es"):
    """A baseline search (ES / TSS / FSS / DS) on one sequence, sharded by
    (pair, block-row band) units balanced by estimated-block count (SURVEY
    8e; config 5's ES is the default line's es_cfg5 leg, any baseline workload
    at N > 1 is strong-scaled this way)."""
    import torch
    import torch.distributed as dist

    import paper_1002_1168_b200 as me
    from paper_1002_1168_b200 import _lib
    from paper_1002_1168_b200 import batch as B
    from paper_1002_1168_b200 import dist as mdist
    from paper_1002_1168_b200 import synth
    import ctypes as C

    cfg_id, algo, bs, S, _ = WORKLOADS[wl]
    F = args.es_frames or {1: 10, 2: 30, 3: 60, 5: 30}[cfg_id]
    pairs, d = F - 2, 2
    luma, alpha = synth.config4_batch_dev(1, BASE_SEED, F, config_id=cfg_id, device=local)
    torch.cuda.synchronize(dev)
    _, _, H, W = luma.shape
    rows, cols = H // bs, W // bs
    cfg = me_config(algo, bs, S)
    n_bands = args.es_bands or (1 if world == 1 else 4)
    units = mdist.band_units(alpha[0], bs, pairs, d, n_bands)
    mine = mdist.split_units(units, world)[rank]
    runs = mdist.unit_runs(mine)
    recs = torch.zeros((1, pairs, rows, cols, 16), dtype=torch.uint8, device=dev)
    stats_acc = torch.zeros((pairs, 6), dtype=torch.int64, device=dev)
    tmp_stats = torch.empty((1, pairs, 48), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    lib = me.lib()
    ctxh = _lib.ctx(local)

    def step():
        stats_acc.zero_()
        for b, p0, p1, r0, r1 in runs:
            n = p1 - p0
            lv, av = luma[:, p0:p1 + d], alpha[:, p0:p1 + d]
            rv, sv = recs[:, p0:p1], tmp_stats[:, :n]
            if n_bands == 1:
                B.run_sequences_dev(cfg, lv, av, rv, sv, device=local, stream=stream.cuda_stream)
            else:
                B.run_band_dev(cfg, lv, av, r0, r1, rv, sv, device=local, stream=stream.cuda_stream)
            stats_acc[p0:p1] += sv[0].view(torch.int64).view(n, 6)
        if world > 1:  # MV words of my units + my partial stats -> rank 0
            cd = mdist.coll_device(dev)
            mvw = mdist.mv_words(recs[0]).to(cd)
            sacc = stats_acc.to(cd)
            outs = [torch.empty_like(mvw) for _ in range(world)] if rank == 0 else None
            sts = [torch.empty_like(sacc) for _ in range(world)] if rank == 0 else None
            dist.gather(mvw, outs, dst=0)
            dist.gather(sacc, sts, dst=0)
            return outs, sts
        return None, None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local).start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.es_steps):
        outs, sts = step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = mdist.max_over_ranks(ev0.elapsed_time(ev1), dev) / args.es_steps
    # search-stage time of this rank's calls (stage events, untimed pass)
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 1))
    stage = (C.c_float * 4)()
    search_ms = 0.0
    for b, p0, p1, r0, r1 in runs:
        n = p1 - p0
        lv, av = luma[:, p0:p1 + d], alpha[:, p0:p1 + d]
        if n_bands == 1:
            B.run_sequences_dev(cfg, lv, av, recs[:, p0:p1], tmp_stats[:, :n], device=local, stream=stream.cuda_stream)
        else:
            B.run_band_dev(cfg, lv, av, r0, r1, recs[:, p0:p1], tmp_stats[:, :n], device=local, stream=stream.cuda_stream)
        _lib.check(lib.me_b200_ctx_stage_ms(ctxh, stage, 4))
        search_ms += stage[2]
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))
    search_ms = mdist.max_over_ranks(search_ms, dev)
    ipk = C.c_double()
    _lib.check(lib.me_b200_probe_int_peak(ctxh, C.byref(ipk)))
    if world > 1:
        dist.barrier()
    if rank != 0:
        return None
    # whole-sequence results on rank 0
    if world > 1:
        owner = {}
        for r, us in enumerate(mdist.split_units(units, world)):
            for b, p, r0, r1, _ in us:
                owner[(p, b)] = (r, r0, r1)
        mv = torch.zeros((pairs, rows, cols), dtype=torch.int32, device=dev)
        for (p, b), (r, r0, r1) in owner.items():
            mv[p, r0:r1] = outs[r][p, r0:r1]
        st = torch.stack(sts).sum(0).cpu().numpy()
        mvn = mv.cpu().numpy()
        dx, dy = (mvn << 16) >> 16, mvn >> 16
        cmp_total = int(st[:, 0].sum())
    else:
        rn = recs[0].cpu().numpy().view(_lib.rec_dtype()).reshape(pairs, rows, cols)
        dx, dy = rn["dx"].astype(np.int32), rn["dy"].astype(np.int32)
        st = stats_acc.cpu().numpy()
        cmp_total = int(st[:, 0].sum())
    ops = cmp_total * bs * bs
    units_mb = pairs * (W // 16) * (H // 16)
    # parity: ES at 4K — sampled estimated blocks spread over the pairs vs the
    # reference's full_search (the whole sequence takes minutes on the host);
    # the other searches — the whole sequence's MV fields + stats vs the reference
    import oracle as O

    lh, ah = luma[0].cpu().numpy(), alpha[0].cpu().numpy()
    parity = None
    if not args.no_parity and not (algo == "ES" and cfg_id == 5):
        rr = np.zeros((1, pairs, rows, cols), _lib.rec_dtype())
        rr["dx"], rr["dy"] = dx, dy  # (half-pel, as the records)
        sn = np.ascontiguousarray(st.astype(np.int64)).view(_lib.stats_dtype()).reshape(1, pairs)
        parity, _ = digest_parity(rr, sn, lh[None], ah[None], cfg_id, algo, bs, S, os.cpu_count() or 1)
    elif not args.no_parity:
        orc = O.Oracle("reference" if O.available("reference") else "port")
        rng = np.random.default_rng(5)
        bad, n_chk = 0, 0
        for p in rng.choice(pairs, size=min(8, pairs), replace=False):
            types = orc.classify(ah[p + d], bs)
            est = np.flatnonzero(types != 0)
            for gi in rng.choice(est, size=min(6, est.size), replace=False):
                v, h = divmod(int(gi), cols)
                (rdx, rdy), rcmp, rcost = orc.block_search(0, lh[p + d], lh[p], h * bs, v * bs, bs, S)
                n_chk += 1
                bad += (int(dx[p, v, h]), int(dy[p, v, h])) != (rdx, rdy)
        parity = {"blocks_checked": n_chk, "mismatches": bad, "how": f"ES MVs of randomly sampled estimated blocks vs the reference's full_search ({orc.kind})"}
    threads = os.cpu_count() or 1
    v_cpu, sample, dt, kind = cpu_sample(wl, lh[None], ah[None], threads)
    peak = ipk.value / 1e12
    ach = ops / (search_ms / 1e3) / 1e12
    return {
        "workload": f"{wl}: BASELINE config {cfg_id} ({GEOMETRY[cfg_id]} x {F}f, {pairs} pairs), {algo} S={S} bs={bs}" + (f", (pair, row-band) units over {world} GPUs" if world > 1 else ""),
        "metric": "macroblocks/sec", "value": units_mb / (ms / 1e3), "unit": "MB/s", "ms_per_step": ms, "steps": args.es_steps,
        "sad_byte_ops_per_step": ops, "search_ms": search_ms,
        "roofline": {"bound": "int", "kernel": f"{'es_kernel' if algo == 'ES' else 'ring_kernel'} (search stage)", "achieved": ach, "peak": peak, "unit": "T byte-ops/s", "frac": ach / peak,
                     "peak_source": "VABSDIFF4.U8.ACC microbenchmark measured in this run on this GPU (me_b200_probe_int_peak)",
                     "note": "achieved = oracle-exact comparisons x 256 byte-ops / search-stage time (CUDA events)"},
        "clocks": clk, "parity": parity,
        "cpu_baseline": {"value": v_cpu, "unit": "MB/s", "cores": threads, "kind": kind, "sample": sample, "seconds": dt},
        "units": {"n": len(units), "bands": n_bands, "per_rank": [len(u) for u in mdist.split_units(units, world)]},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4-pa", choices=sorted(WORKLOADS))
    ap.add_argument("--n-seq", type=int, default=0, help="config 4: sequences in total (strong) or per rank (--weak)")
    ap.add_argument("--weak", action="store_true", help="config 4: every rank runs its own batch")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-es", action="store_true", help="skip the es_cfg5 leg of the default run")
    ap.add_argument("--no-bits", action="store_true", help="skip the bit-packed-mask layout leg")
    ap.add_argument("--no-critical", action="store_true", help="skip the single-sequence critical-path leg")
    ap.add_argument("--es-steps", type=int, default=5)
    ap.add_argument("--es-frames", type=int, default=0)
    ap.add_argument("--es-bands", type=int, default=0, help="ES block-row bands per pair (default 1 on one GPU, 4 on several)")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"], help="gloo: host collectives (tests)")
    ap.add_argument("--same-device", action="store_true", help="test switch: every rank uses cuda:0 (with --dist-backend gloo)")
    args = ap.parse_args()
    wl = args.workload
    if args.impl == "reference":
        return run_reference_arm(args, wl)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return respawn_torchrun(sys.argv[1:], args.gpus)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if args.same_device:  # test switch: every rank on cuda:0 (gloo collectives through the host)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    # baseline searches (ES / TSS / FSS / DS) on several GPUs: (pair, row-band) units, strong-scaled
    units_line = wl == "cfg5-es" or (WORKLOADS[wl][1] != "PA" and world > 1)
    line = bench_pa_batch(args, wl, world, rank, local, dev) if not units_line else None
    es = None
    if units_line or (wl == "cfg4-pa" and not args.no_es):
        es = bench_units(args, world, rank, local, dev, wl if units_line else "cfg5-es")
    if rank == 0:
        if line is None:  # the units leg is the line
            line = {"metric": "macroblocks/sec", "value": es["value"], "unit": "MB/s", "n_gpus": world, "steps": es["steps"], "warmup": max(args.warmup, 3),
                    "ms_per_step": es["ms_per_step"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
                    "data": "synthetic (seeded integer config generator, SURVEY §8d)", "config": {"workload": es["workload"]}, "roofline": es["roofline"],
                    "cpu_baseline": es["cpu_baseline"], "e2e": None, "clocks": es["clocks"], "parity": es["parity"]}
        else:
            line["es_cfg5"] = es
            if wl == "cfg4-pa" and not args.no_critical and world == 1:
                line["critical_path"] = bench_critical_path(args, local, dev)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
