#!/usr/bin/env python3
"""Benchmark of the B200 shape-adaptive motion-estimation hot path.

Default workload (BASELINE.json config 4, the throughput batch): per GPU, 256
independent CIF 352x288 sequences x 30 frames from the config-2 generator
(seed = base + i), proposed algorithm (PA: BRS + PRS) at +/-16, 8x8 blocks,
ref_distance 2, plus motion compensation and PSNR for every pair.  One "step"
= one pass of the whole pipeline (classify -> wavefront sort -> PA -> MC+PSNR)
over the batch.  Metric: macroblocks/s = (W/16)(H/16) x pairs x sequences / s,
every 16x16 macroblock counted (transparent ones included).

  python bench.py [--gpus N --steps K --warmup W] [--workload cfg4-pa|cfg5-es|...]
  python bench.py --impl reference ...   # the reference's own CPU code path

N > 1 (torchrun): every rank runs its own 256-sequence batch (weak scaling; seeds
base + 256 * rank + i), no data-path collective; the motion-vector fields of
each step are gathered into rank 0 over NCCL inside the timed region (the
north star's "final gather of MV fields over NVLink"): packed as int8 (dx, dy)
pairs when S <= 63 and gathered asynchronously while the next step computes
(paper_1002_1168_b200/dist.py FieldGatherer); the last gather completes before
the closing event.  --strong shards one
256-sequence batch across ranks instead.
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

# workload -> (config id, algo, block size, search range, default sequences per GPU)
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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def int_peak_path():
    return os.path.join(ROOT, "profiles", "int_peak.json")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50", "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def gen_inputs(cfg_id, n_seq, first_seed, frames=None, out_luma=None, out_alpha=None):
    from paper_1002_1168_b200 import synth

    if cfg_id == 4:
        return synth.config4_batch(n_seq, first_seed, frames, out_luma, out_alpha, threads=min(32, os.cpu_count() or 8))
    l, a = synth.config_sequence(cfg_id, first_seed, frames)
    if out_luma is not None:
        out_luma[0] = l
        out_alpha[0] = a
        return out_luma, out_alpha
    return l[None], a[None]


def me_config(algo, bs, S):
    import paper_1002_1168_b200 as me

    return me.BatchConfig(algo=me.Algo[algo], search=me.SearchConfig(search_range=S, block_size=bs, ref_distance=2), prs=me.PrsConfig())


# ---------------------------------------------------------------------------
# CPU legs (reference arm and cpu_baseline): the reference's own code path
# (oracle/_ref/libme_ref.so, compiled from the unmodified sources) when built,
# else the oracle port.


def cpu_oracle():
    import oracle

    if oracle.available("reference"):
        return oracle.Oracle("reference"), "reference"
    if not oracle.available("port"):
        oracle.build(ref=False)
    return oracle.Oracle("port"), "port"


def cpu_measure(wl, luma, alpha, threads, max_seq=0):
    """Times the CPU implementation on a bounded sample; returns (MB/s, sample, seconds)."""
    import oracle as O

    cfg_id, algo, bs, S, _ = WORKLOADS[wl]
    orc, kind = cpu_oracle()
    cfg = O.make_cfg(algo=ALGO_ID[algo], search_range=S, block_size=bs, ref_distance=2)
    n_seq, F, H, W = luma.shape
    mb_per_pair = (W // 16) * (H // 16)
    if algo == "PA" or algo in ("TSS", "FSS", "DS"):
        if algo == "PA":
            # one sequence per thread at a time (pairs chain through the temporal candidate)
            n = min(n_seq, max_seq or max(threads, 1) * 2)
            t = time.perf_counter()
            orc.time_sequences(cfg, np.ascontiguousarray(luma[:n]), np.ascontiguousarray(alpha[:n]), threads)
            dt = time.perf_counter() - t
            return n * (F - 2) * mb_per_pair / dt, f"{n} sequences x {F - 2} pairs ({kind}, {threads} threads)", dt, kind
        n_pairs = F - 2
        t = time.perf_counter()
        orc.time_pairs(cfg, luma[0], alpha[0], 0, n_pairs, threads)
        dt = time.perf_counter() - t
        return n_pairs * mb_per_pair / dt, f"1 sequence x {n_pairs} pairs ({kind}, {threads} threads)", dt, kind
    # ES: bounded sample of estimated blocks of the first pair(s); rate in
    # macroblocks/s of the full workload = sample blocks/s scaled by the
    # all-block / estimated-block ratio of that pair
    types = orc.classify(alpha[0, 2], bs)
    cols = W // bs
    est = np.flatnonzero(types != 0)
    if est.size == 0:
        return None, "no estimated blocks", 0.0, kind
    # sample ~ (threads * 4) blocks, spread over the frame
    k = min(est.size, max(threads * 4, 16))
    pick = est[np.linspace(0, est.size - 1, k).astype(int)]
    xy = np.stack([(pick % cols) * bs, (pick // cols) * bs], 1).astype(np.int32)
    t = time.perf_counter()
    orc.time_blocks(cfg, np.ascontiguousarray(luma[0, 2]), np.ascontiguousarray(luma[0, 0]), xy, threads)
    dt = time.perf_counter() - t
    blocks_per_s = k / dt
    # a pair's macroblocks are done when its estimated blocks are
    mbs = blocks_per_s * mb_per_pair / est.size
    return mbs, f"{k} of {est.size} estimated blocks of pair 0 ({kind}, {threads} threads), scaled to whole pairs", dt, kind


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg_id, algo, bs, S, nseq = WORKLOADS[wl]
    threads = os.cpu_count() or 1
    n = nseq if cfg_id == 4 else 1
    n_gen = min(n, max(64, 4 * threads)) if cfg_id == 4 else 1
    luma, alpha = gen_inputs(cfg_id, n_gen, BASE_SEED)
    vals = []
    for i in range(args.warmup + args.steps):
        v, sample, dt, kind = cpu_measure(wl, luma, alpha, threads, max_seq=max(64, 4 * threads))
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference",
        "metric": "macroblocks/sec",
        "value": value,
        "unit": "MB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (seeded config generator, SURVEY §8d)",
        "config": workload_config(wl, args),
        "cpu_baseline": {"value": value, "unit": "MB/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "MB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(wl, args):
    cfg_id, algo, bs, S, nseq = WORKLOADS[wl]
    geo = {1: "QCIF 176x144 x 10f", 2: "CIF 352x288 x 30f", 3: "1920x1088 x 60f", 4: "CIF 352x288 x 30f", 5: "3840x2160 x 30f"}[cfg_id]
    return {
        "workload": f"{wl}: BASELINE config {cfg_id} ({geo}), {algo} S={S} bs={bs}, ref_distance 2" + (f", {args.n_seq or nseq} sequences/GPU" if cfg_id == 4 else ""),
        "config_id": cfg_id,
        "algo": algo,
        "search_range": S,
        "block_size": bs,
        "sequences_per_gpu": (args.n_seq or nseq),
        "l2": "inputs larger than L2 (126 MB)" if cfg_id in (3, 4, 5) else "L2 flushed between steps (256 MB write)",
        "parallelism": f"sequences sharded, {args.gpus} GPU(s), MV-field gather to rank 0 (int8 pairs for S <= 63, overlapped with the next step)",
    }


# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4-pa", choices=sorted(WORKLOADS))
    ap.add_argument("--n-seq", type=int, default=0, help="sequences per GPU (config 4)")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--strong", action="store_true", help="shard one batch across ranks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    args = ap.parse_args()
    wl = args.workload
    if args.impl == "reference":
        return run_reference_arm(args, wl)

    import torch
    import torch.distributed as dist

    import paper_1002_1168_b200 as me
    from paper_1002_1168_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg_id, algo, bs, S, nseq_default = WORKLOADS[wl]
    n_seq = args.n_seq or nseq_default
    if args.strong and cfg_id == 4:
        n_seq = (n_seq + world - 1) // world
    warmup = max(args.warmup, 3)
    frames = args.frames or None

    # inputs: generated on the host into pinned memory, then made resident
    from paper_1002_1168_b200 import synth

    p0 = synth.preset(cfg_id, BASE_SEED, frames)
    F, H, W = p0.frames, p0.height, p0.width
    # generated on the GPU (me_b200_synth_dev, byte-identical to the host
    # generator), then copied to pinned host memory for the e2e and CPU legs
    t0 = time.perf_counter()
    luma, alpha = synth.config4_batch_dev(n_seq, BASE_SEED + 256 * rank, frames, config_id=cfg_id, device=local)
    torch.cuda.synchronize(dev)
    pin = torch.empty((2, n_seq, F, H, W), dtype=torch.uint8, pin_memory=True)
    pin[0].copy_(luma)
    pin[1].copy_(alpha)
    hl, ha = pin[0].numpy(), pin[1].numpy()
    log(f"[rank {rank}] generated {n_seq} x {F} x {H}x{W} on the device in {time.perf_counter() - t0:.2f}s")
    cfg = me_config(algo, bs, S)
    pairs = F - 2
    rows, cols = H // bs, W // bs
    recs = torch.empty((n_seq, pairs, rows, cols, 16), dtype=torch.uint8, device=dev)
    stats = torch.empty((n_seq, pairs, 48), dtype=torch.uint8, device=dev)
    from paper_1002_1168_b200 import dist as mdist

    gatherer = mdist.FieldGatherer(S) if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if cfg_id in (1, 2) else None
    stream = torch.cuda.current_stream(dev)
    lib = me.lib()
    ctxh = _lib.ctx(local)
    # stage events only in the untimed breakdown pass: an event between two
    # launches would also break their programmatic-dependent-launch chain
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))
    import ctypes as C

    stage = (C.c_float * 4)()
    stage_sum = np.zeros(4)

    def step(stages):
        me.run_sequences_dev(cfg, luma, alpha, recs, stats, device=local, stream=stream.cuda_stream)
        if stages:  # waits for the step: only in the untimed breakdown pass below
            _lib.check(lib.me_b200_ctx_stage_ms(ctxh, stage, 4))
            stage_sum[:] += np.array(stage[:])
        if gatherer is not None:  # step k's packed MV field -> rank 0, overlapping step k+1
            gatherer.submit(recs)
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
    clocks = ClockSampler(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(False)
    if gatherer is not None:
        gatherer.finish()  # the last step's gather completes inside the timed region
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    from paper_1002_1168_b200 import batch as B

    launches_per_step = B.last_launches(local)
    # per-stage breakdown (CUDA events on the launching stream), untimed
    n_stage = min(args.steps, 20)
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 1))
    for _ in range(n_stage):
        step(True)
    _lib.check(lib.me_b200_ctx_set_profiling(ctxh, 0))  # the e2e leg runs without stage events
    if gatherer is not None:
        gatherer.finish()
    stage_sum *= args.steps / n_stage
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    total_units = n_seq * pairs * (W // 16) * (H // 16) * world
    value = total_units / (ms_per_step / 1e3)

    # correctness guard: the bench result of sequence 0 equals a host-API run
    hrec = recs[0].cpu().numpy().view(_lib.rec_dtype()).reshape(pairs, rows, cols)
    hstat = stats.cpu().numpy().view(_lib.stats_dtype()).reshape(n_seq, pairs)

    # roofline of the step (HBM): every luma + alpha byte read once, records written once
    hbm_peak, peak_src = peaks()
    stage_ms = stage_sum / args.steps
    alg_bytes = n_seq * F * W * H * 2 + n_seq * pairs * rows * cols * 16
    pipe_ms = float(stage_ms.sum())
    roof = None
    # dram bytes per step from the committed ncu --set full captures (profiles/ncu_traffic.json)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(args.workload)
        if tr and tr.get("n_seq") == n_seq:
            traffic, traffic_src = float(sum(tr["dram_bytes"].values())), tr
    if algo == "PA":
        ach = alg_bytes / (pipe_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": f"pipeline classify+scan+fill+PA wavefront search ({launches_per_step} launches/step)", "achieved": ach, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic, "traffic_by_kernel": traffic_src["dram_bytes"] if traffic_src else None, "algorithmic_bytes_per_step": alg_bytes, "pipeline_ms": pipe_ms,
                "dominant": {"kernel": "pa_fast + pa_quad + pa_fast (wavefront search)", "ms": float(stage_ms[2]), "share": float(stage_ms[2]) / pipe_ms, "bound": "dependency latency + issue (see DESIGN.md)"}}
    else:
        cmp_total = int(hstat["block_comparisons"].sum())
        ops = cmp_total * bs * bs  # SAD byte-ops of the search stage
        search_s = stage_ms[2] / 1e3
        ip = None
        if os.path.exists(int_peak_path()):
            with open(int_peak_path()) as f:
                ip = json.load(f)
        peak_t = ip["byte_ops_per_s"] / 1e12 if ip else None
        ach = ops / search_s / 1e12
        roof = {"bound": "int", "kernel": f"{algo.lower()}_kernel (search stage)", "achieved": ach, "peak": peak_t, "peak_source": "profiles/int_peak.json (VABSDIFF4 microbenchmark)" if ip else "not measured", "unit": "T byte-ops/s", "frac": (ach / peak_t) if peak_t else None, "traffic": None, "sad_byte_ops_per_step": ops, "search_ms": float(stage_ms[2])}

    # end to end through the public host-pointer C ABI: pinned H2D + pipeline + D2H
    e2e = None
    if not args.no_e2e:
        hrecs = torch.empty((n_seq, pairs, rows, cols, 16), dtype=torch.uint8, pin_memory=True)
        hstats = torch.empty((n_seq, pairs, 48), dtype=torch.uint8, pin_memory=True)
        from paper_1002_1168_b200 import batch as B

        n_e2e = args.e2e_steps or max(1, min(args.steps, 10))
        B.run_sequences_ptr(cfg, n_seq, F, W, H, hl.ctypes.data, ha.ctypes.data, hrecs.data_ptr(), hstats.data_ptr(), local)  # warm
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(n_e2e):
            B.run_sequences_ptr(cfg, n_seq, F, W, H, hl.ctypes.data, ha.ctypes.data, hrecs.data_ptr(), hstats.data_ptr(), local)
        e2e_s = (time.perf_counter() - t) / n_e2e
        if world > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        if not np.array_equal(hrecs.numpy()[0].view(_lib.rec_dtype()).reshape(pairs, rows, cols), hrec):
            raise SystemExit("e2e records differ from the device-resident run")
        h2d, d2h = B.last_transfer_bytes(local)  # counted by the library: alpha masks cross bit-packed
        # this box's pinned H2D bandwidth (256 MiB copies): the e2e step's copy floor is h2d / it
        probe_h = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        probe_d = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        probe_d.copy_(probe_h, non_blocking=True)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(4):
            probe_d.copy_(probe_h, non_blocking=True)
        ev1.record()
        torch.cuda.synchronize()
        h2d_gbs = 4 * (256 << 20) / (ev0.elapsed_time(ev1) * 1e-3) / 1e9
        del probe_h, probe_d
        e2e = {"value": total_units / e2e_s, "unit": "MB/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": n_e2e, "s_per_step": e2e_s,
               "input_bytes_per_step": int(2 * n_seq * F * W * H), "h2d_gbs_measured": h2d_gbs, "h2d_floor_ms": h2d / h2d_gbs / 1e6, "note": "pinned host buffers; luma as bytes, binary alpha bit-packed on the host cores (AVX-512) with all-zero 64-pixel words elided, expanded on the GPU"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        # the whole batch (~10 CPU-seconds at 256 sequences)
        v, sample, dt, kind = cpu_measure(wl, hl, ha, threads, max_seq=n_seq)
        cpu = {"value": v, "unit": "MB/s", "cores": threads, "kind": kind, "sample": sample, "seconds": dt}

    if rank == 0:
        est = int(hstat["blocks_opaque"].sum() + hstat["blocks_boundary"].sum())
        line = {
            "metric": "macroblocks/sec",
            "value": value,
            "unit": "MB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic (seeded integer config generator, SURVEY §8d; no public sequences in this container)",
            "config": workload_config(wl, args),
            "roofline": roof,
            "stages_ms": {"classify": stage_ms[0], "sort": stage_ms[1], "search": stage_ms[2], "mc_psnr": stage_ms[3]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "estimated_blocks_per_gpu": int(est * 1),
            "macroblocks_per_step": int(total_units),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
