#!/usr/bin/env python
"""bench.py -- LASNet coarse-grained spatially-dynamic residual block on B200.

Workload (BASELINE.json configs[1]): ResNet-50 stage-3
identity bottleneck (He et al. conv3_x; LASNet stage 2), N = 128 images per GPU,
28x28x512 NHWC bf16, c_mid = 128, granularity S = 4, activation rate r ~ 0.5
(masker bias calibrated on a separate batch), synthetic seeded inputs, random-
init weights.  A step = one pass of the whole hot path (masker -> compaction ->
gather+conv1 -> conv2 -> conv3+scatter-add) over the batch, in place.

Timing: W warm-up steps, then exactly K timed steps bracketed by barrier +
synchronize; CUDA events on the launching stream around every step; before
each step (untimed) the input is restored and L2 is flushed by reading a
256 MiB buffer (x is 103 MB < 126 MB L2).  Multi-GPU (torchrun): weak scaling,
each rank its own 128 images, no data-path collective; max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lasnet|reference]
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

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LASNet-R101 images/s & dyn-block latency vs activation rate (1/2/4/8 B200)"
WORKLOAD = dict(n=128, h=28, w=28, c_in=512, c_mid=128, s=4, r=0.5)
WORKLOAD_NAME = "resnet50-stage3 identity dyn-block (BASELINE configs[1]) N=128/GPU 28x28x512 c_mid=128 S=4 r=0.5"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="lasnet", choices=["lasnet", "reference"])
    ap.add_argument("--s", type=int, default=WORKLOAD["s"])
    ap.add_argument("--r", type=float, default=WORKLOAD["r"])
    ap.add_argument("--n", type=int, default=WORKLOAD["n"])
    ap.add_argument("--hw", type=int, default=WORKLOAD["h"], help="(experiments) spatial size of the block")
    ap.add_argument("--c-in", type=int, default=WORKLOAD["c_in"], help="(experiments) block width")
    ap.add_argument("--c-mid", type=int, default=WORKLOAD["c_mid"], help="(experiments) bottleneck width")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--detail", default=None, help="write per-kernel detail JSON here")
    ap.add_argument("--network", type=int, default=1, help="1: also time the LAS-ResNet-101 forward (BASELINE "
                                                             "configs[2]: 224x224, global batch 256 split over the ranks)")
    ap.add_argument("--graph", type=int, default=1, help="1: time CUDA-graph replays of the step (captured once on "
                                                          "the same buffers), 0: eager launches")
    ap.add_argument("--schedule", default="auto", choices=["auto", "separate", "fused"],
                    help="separate: north-star branch (masker, then gather+conv1 on halos); fused: the paper's "
                         "Table-1 schedule (masker fused into a static conv1); auto: lasnet_choose_schedule(r)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 10:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [r for r in rows if r[4] not in ("0", "[N/A]")] or rows
        sm = [float(r[1]) for r in load if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in load:
            for nm, v in zip(names, r[6:10]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(load)}


# ------------------------------------------------------ algorithmic work ----

def algorithmic_work(mask_cells: np.ndarray, n, h, w, c_in, c_mid, c_out, s):
    """Per-kernel algorithmic bytes and FLOPs for the concrete mask (DESIGN.md
    "Roofline accounting"; SURVEY 8(d) per-unit figures)."""
    gh, gw = -(-h // s), -(-w // s)
    ids = np.flatnonzero(mask_cells.reshape(-1))
    P = len(ids)
    g = ids % (gh * gw)
    gy, gx = g // gw, g % gw
    # in-image halo pixels of each active patch: (S+2)^2 window at (gy*S-1, gx*S-1)
    y0, x0 = gy * s - 1, gx * s - 1
    hy = np.minimum(y0 + s + 2, h) - np.maximum(y0, 0)
    hx = np.minimum(x0 + s + 2, w) - np.maximum(x0, 0)
    halo_px = int(np.sum(hy * hx))
    oy = np.minimum(gy * s + s, h) - gy * s
    ox = np.minimum(gx * s + s, w) - gx * s
    out_px = int(np.sum(oy * ox))
    e = 2
    hs2, ss = (s + 2) ** 2, s * s
    W1, W2, W3 = c_mid * c_in * e, 9 * c_mid * c_mid * e, c_out * c_mid * e
    k = {
        "mask_compact": dict(bytes=n * h * w * c_in * e + n * gh * gw + 4 * P + 4, flops=2 * n * h * w * c_in),
        # fused steps 4+5: h1 read once per tap-row window, residual + y, both weights
        "conv23": dict(bytes=P * hs2 * c_mid * e + 2 * out_px * c_out * e + 9 * c_mid * c_mid * e + c_out * c_mid * e,
                       flops=2 * out_px * 9 * c_mid * c_mid + 2 * out_px * c_mid * c_out),
        "conv1": dict(bytes=halo_px * c_in * e + P * hs2 * c_mid * e + W1, flops=2 * halo_px * c_in * c_mid),
        "conv2": dict(bytes=P * hs2 * c_mid * e + P * ss * c_mid * e + W2, flops=2 * out_px * 9 * c_mid * c_mid),
        "conv3": dict(bytes=P * ss * c_mid * e + 2 * out_px * c_out * e + W3, flops=2 * out_px * c_mid * c_out),
        # masker-fused schedule: dense conv1 + masker partials; decision + compaction + h1 halo gather
        "conv1_mask": dict(bytes=n * h * w * (c_in * e + c_mid * e + 16) + W1,
                           flops=2 * n * h * w * c_in * (c_mid + 1)),
        "decide_gather": dict(bytes=n * h * w * 16 + n * gh * gw + 4 * P + halo_px * c_mid * e + P * hs2 * c_mid * e,
                              flops=0),
    }
    block = dict(
        bytes=n * h * w * c_in * e + n * gh * gw + 4 * P + halo_px * c_in * e + 2 * out_px * c_out * e + W1 + W2 + W3,
        flops=k["conv1"]["flops"] + k["conv2"]["flops"] + k["conv3"]["flops"])
    # the masker-fused schedule's own minimum: x once, h1 written once and its halos
    # read back, residual + y of active pixels, weights; dense conv1 FLOPs
    block_fused = dict(
        bytes=n * h * w * (c_in + c_mid) * e + n * gh * gw + 4 * P + halo_px * c_mid * e + 2 * out_px * c_out * e
        + W1 + W2 + W3,
        flops=2 * n * h * w * c_in * c_mid + k["conv2"]["flops"] + k["conv3"]["flops"])
    dense = dict(bytes=2 * n * h * w * c_in * e + W1 + W2 + W3,
                 flops=2 * n * h * w * (c_in * c_mid + 9 * c_mid * c_mid + c_mid * c_out))
    return k, block, dense, dict(P=P, halo_px=halo_px, out_px=out_px, r_patch=P / (n * gh * gw),
                                 r_pixel=out_px / (n * h * w), block_fused=block_fused)


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the latest committed
    ncu --set full capture (profiles/ncu_full_<tag>.json), or (None, None)."""
    import glob

    names = {"mask_compact": "mask_compact", "conv1": "conv1_dyn", "conv2": "conv2_dyn", "conv3": "conv3_dyn",
             "conv23": "conv23_dyn", "conv1_mask": "conv1_mask", "decide_gather": "decide_gather"}
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_*.json")))  # by round tag
    for f in reversed(files):
        d = json.load(open(f))
        for e in d.get("full", []):
            if e.get("kernel") == names.get(kernel):
                return int(e.get("dram_read", 0) + e.get("dram_write", 0)), os.path.relpath(f, ROOT)
    return None, None


def roofline_entry(work, ms, hbm, tfl):
    t_hbm = work["bytes"] / (hbm * 1e9)
    t_tc = work["flops"] / (tfl * 1e12)
    if t_hbm >= t_tc:
        ach = work["bytes"] / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4)}
    ach = work["flops"] / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": tfl, "unit": "TFLOP/s", "frac": round(ach / tfl, 4)}


# ------------------------------------------------------------ cpu oracle ----

def oracle_sample(x_cpu, wts_cpu, wm_cpu, bm, s, k_images, threads):
    """The oracle as it stands, run on the first k images: masker -> compact ->
    literal gather/conv/scatter block.  Returns seconds."""
    import oracle
    import synth

    oracle.set_threads(threads)
    xd = synth.to_f64(x_cpu[:k_images])
    wd = synth.weights_f64(wts_cpu)
    t0 = time.perf_counter()
    m, _ = oracle.masker(xd, synth.to_f64(wm_cpu), bm, s)
    idx, _ = oracle.compact(m)
    oracle.dyn_block_literal(xd, wd, idx, s)
    return time.perf_counter() - t0


def cpu_baseline(x_cpu, wts_cpu, wm_cpu, bm, s, budget_s, n_total):
    import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    t1 = oracle_sample(x_cpu, wts_cpu, wm_cpu, bm, s, 2, threads)
    k = int(max(2, min(n_total, budget_s / max(t1 / 2, 1e-6))))
    t = oracle_sample(x_cpu, wts_cpu, wm_cpu, bm, s, k, threads) if k > 2 else t1
    return {"value": round(k / t, 2), "unit": "images/s", "cores": threads, "kind": "oracle",
            "sample": f"first {k} of the {n_total} images, same S/weights/masker bias, fp64 literal mode "
                      f"(masker+compact+gather/conv/scatter), OpenMP over patches; {t:.2f} s"}


# ------------------------------------------------------------- reference ----

def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (this tier's
    reference arm), each step a bounded sample of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth

    oracle.build()
    wl = dict(WORKLOAD, n=args.n, s=args.s, r=args.r)
    x = synth.make_x(wl["n"], wl["h"], wl["w"], wl["c_in"], seed=0)
    wts = synth.make_block_weights(wl["c_in"], wl["c_mid"], wl["c_in"], seed=1)
    wm = synth.make_masker_weights(wl["c_in"], seed=2)
    xc = synth.make_x(wl["n"], wl["h"], wl["w"], wl["c_in"], seed=1000)
    _, l0 = oracle.masker(synth.to_f64(xc), synth.to_f64(wm), 0.0, wl["s"])
    lg = np.sort(l0.reshape(-1))
    kk = int(round(wl["r"] * lg.size))
    bm = float(np.float32(-0.5 * (lg[lg.size - kk - 1] + lg[lg.size - kk])))
    threads = os.cpu_count() or 1
    t1 = oracle_sample(x, wts, wm, bm, wl["s"], 2, threads)
    k_img = int(max(2, min(wl["n"], 3.0 / max(t1 / 2, 1e-6))))
    for _ in range(args.warmup):
        oracle_sample(x, wts, wm, bm, wl["s"], k_img, threads)
    ts = [oracle_sample(x, wts, wm, bm, wl["s"], k_img, threads) for _ in range(args.steps)]
    tot = sum(ts)
    val = k_img * args.steps / tot
    line = {"metric": METRIC, "value": round(val, 3), "unit": "images/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME, "global_batch": wl["n"], "sample_images_per_step": k_img,
                       "S": wl["s"], "r_target": wl["r"]},
            "cpu_baseline": {"value": round(val, 3), "unit": "images/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {k_img} of {wl['n']} images per step"},
            "e2e": {"value": round(val, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- lasnet ----

def run_lasnet(args):
    import torch.distributed as dist

    import synth
    import paper_2210_06223_b200 as L
    from paper_2210_06223_b200 import _lib, build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0 or not os.path.exists(_lib.LIB_PATH):
        build.build()
    if world > 1:
        dist.barrier()
    lib = _lib.load()

    wl = dict(WORKLOAD, n=args.n, s=args.s, r=args.r, h=args.hw, w=args.hw, c_in=args.c_in, c_mid=args.c_mid)
    n, h, w, c_in, c_mid, s = (wl[k] for k in ("n", "h", "w", "c_in", "c_mid", "s"))
    x_cpu = synth.make_x(n, h, w, c_in, seed=0 + 7919 * rank)
    wts_cpu = synth.make_block_weights(c_in, c_mid, c_in, seed=1)
    wm_cpu = synth.make_masker_weights(c_in, seed=2)
    if args.schedule == "auto":
        sched = L.choose_schedule(n, h, w, c_in, c_mid, c_in, s, wl["r"])
    else:
        sched = L.SCHED_FUSED if args.schedule == "fused" else L.SCHED_SEPARATE
    sched_name = "fused" if sched == L.SCHED_FUSED else "separate"
    # separate: the step-by-step north-star calls (mask_compact + dyn_block); fused: lasnet_block_forward
    blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts_cpu, wm_cpu, 0.0,
                     schedule=L.SCHED_FUSED if sched == L.SCHED_FUSED else None)
    # masker bias calibrated on a separate batch of the same distribution
    blk.calibrate_bias(synth.make_x(n, h, w, c_in, seed=1000 + rank).cuda(), wl["r"])
    x = x_cpu.cuda()
    y = torch.empty_like(x)
    y2 = torch.empty_like(x)
    # L2 flush by READING 256 MiB (> 126 MB L2): leaves L2 full of clean lines, so
    # the timed step does not pay for write-backs of the flush itself
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()

    def flush_l2():
        flush.sum()

    def prep():
        y.copy_(x)
        flush_l2()

    for _ in range(max(args.warmup, 3)):
        prep()
        blk.forward(y)
    torch.cuda.synchronize()
    mask_cells = blk.mask_buf.cpu().numpy()
    kwork, bwork, dwork, stats = algorithmic_work(mask_cells, n, h, w, c_in, c_mid, c_in, s)

    K = args.steps
    fused23 = os.environ.get("LASNET_NO_FUSE", "0") != "1" and c_mid in (64, 128) and c_in % 64 == 0 and 192 <= c_in <= 512
    head = ["conv1_mask", "decide_gather"] if sched == L.SCHED_FUSED else ["mask_compact", "conv1"]
    names = head + (["conv23"] if fused23 else ["conv2", "conv3"])
    ev_step = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    ev_k = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * len(names))] for _ in range(K)]
    for row in ev_k:
        for e in row:
            e.record(stream)  # materialise the cudaEvent_t handles
    handles = [ctypes_array(row) for row in ev_k]

    step_fn = lambda: blk.forward(y)  # noqa: E731
    l0 = blk.launches
    prep()
    blk.forward(y)  # one eager step: the kernels one step launches (a graph replays exactly these)
    n_launch = blk.launches - l0
    if args.graph:
        graph = blk.capture(y)
        step_fn = graph.replay
        for _ in range(2):
            prep()
            step_fn()

    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = blk.launches
    # headline: CUDA events around each step only (per-kernel events would
    # serialise the programmatic-dependent launches between the kernels)
    for k in range(K):
        prep()
        ev_step[k][0].record(stream)
        step_fn()
        ev_step[k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = blk.launches - launches0 if not args.graph else n_launch * K
    step_ms = [a.elapsed_time(b) for a, b in ev_step]
    tot_ms = sum(step_ms)
    # breakdown pass (same steps, not the headline): events around every kernel
    for k in range(K):
        prep()
        lib.lasnet_set_kernel_events(handles[k], len(names))
        blk.forward(y)
    lib.lasnet_set_kernel_events(None, 0)
    torch.cuda.synchronize()
    kern_ms = {nm: statistics.fmean(ev_k[k][2 * i].elapsed_time(ev_k[k][2 * i + 1]) for k in range(K))
               for i, nm in enumerate(names)}

    # dense comparator: the same kernels on every pixel (lasnet_dense_block)
    for _ in range(3):
        flush_l2()
        blk.dense(x, y2)
    dense_ms = []
    for k in range(K):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        blk.dense(x, y2)
        b.record(stream)
        dense_ms.append((a, b))
    torch.cuda.synchronize()
    dense_ms = [a.elapsed_time(b) for a, b in dense_ms]

    # end to end through the public API with pinned HOST buffers
    x_host = x_cpu.pin_memory()
    y_host = torch.empty_like(x_cpu).pin_memory()
    for _ in range(2):
        blk.forward_host(x_host, y_host, y)
    e2e_ev = []
    for k in range(K):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        blk.forward_host(x_host, y_host, y)
        b.record(stream)
        e2e_ev.append((a, b))
    torch.cuda.synchronize()
    e2e_serial_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
    # the same K steps as a serving loop (DynBlock.stream_host): step i+1's H2D and step
    # i-1's D2H overlap step i (two device buffers, one copy stream per direction)
    y_b = torch.empty_like(y)
    y_host2 = torch.empty_like(x_cpu).pin_memory()
    blk.stream_host([x_host], [y_host, y_host2], [y, y_b], 2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    blk.stream_host([x_host], [y_host, y_host2], [y, y_b], K, before_step=lambda i: flush_l2())
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b)
    clocks = sampler.stop()

    from paper_2210_06223_b200 import dist as ldist

    tot_max, e2e_max, e2e_serial_max, dense_max = ldist.max_over_ranks(
        [tot_ms, e2e_ms, e2e_serial_ms, statistics.fmean(dense_ms)], device="cuda")
    net_info = None
    if args.network:
        err = None
        try:
            nd, nn_, n_loc, nrate = network_measure(world, max(5, min(K, 10)))
        except Exception as e:  # the block headline above stands on its own
            nd = nn_ = float("inf")
            n_loc, nrate, err = 256 // world, 0.0, f"{type(e).__name__}: {e}"[:300]
        # every rank joins the reduction, failed or not (a rank skipping it would hang the others)
        nd_max, nn_max = ldist.max_over_ranks([nd, nn_], device="cuda")
        if err is not None or nd_max == float("inf"):
            net_info = {"error": err or "failed on another rank"}
        else:
            net_info = {"model": "LAS-ResNet-101 (S_net 4-4-2-1, projection blocks static)", "image": "224x224",
                        "global_batch": n_loc * world, "per_gpu_batch": n_loc, "r_target": 0.5,
                        "r_patch_mean": round(nrate, 4), "ms_per_forward": round(nd_max, 4),
                        "images_per_s": round(n_loc * world / (nd_max * 1e-3), 1),
                        "dense_identity_ms_per_forward": round(nn_max, 4),
                        "dense_identity_images_per_s": round(n_loc * world / (nn_max * 1e-3), 1),
                        "speedup_vs_dense": round(nn_max / nd_max, 3),
                        "timing": "CUDA events around one CUDA-graph replay of the whole forward, median, max over ranks"}
    # the exchange step of SURVEY 8(e): summed active-cell statistics and per-rank step times
    act_all, cells_all = ldist.sum_over_ranks([stats["P"], mask_cells.size], device="cuda")
    rank_ms = [t / K for t in ldist.gather_over_ranks(tot_ms, device="cuda")]
    value = ldist.throughput(n, world, K, tot_max)
    e2e_val = ldist.throughput(n, world, K, e2e_max)

    if rank == 0:
        hbm, tfl, tfl_sus, src = peaks()
        dom = max(names, key=lambda nm: kern_ms[nm])
        roof = roofline_entry(kwork[dom], kern_ms[dom], hbm, tfl)
        traffic, tsrc = ncu_traffic(dom)
        roof.update({"kernel": dom, "traffic": traffic, "traffic_source": tsrc, "peak_source": src,
                     "algorithmic": {"bytes": kwork[dom]["bytes"], "flops": kwork[dom]["flops"]},
                     "share_of_step": round(kern_ms[dom] / sum(kern_ms.values()), 3),
                     "timing": "CUDA events around this kernel on its launch stream, breakdown pass"})
        # every kernel of the step against its own bound (north_star: tensor-pipe work for the convolutions,
        # achieved HBM GB/s for the mask / gather / scatter kernels)
        kern_roof = {}
        for nm in names:
            e = roofline_entry(kwork[nm], kern_ms[nm], hbm, tfl)
            e["algorithmic"] = {"bytes": kwork[nm]["bytes"], "flops": kwork[nm]["flops"]}
            if e["bound"] == "hbm" and kwork[nm]["flops"]:
                e["tflops"] = round(kwork[nm]["flops"] / (kern_ms[nm] * 1e-3) / 1e12, 1)
            kern_roof[nm] = e
        blk_roof = roofline_entry(bwork, statistics.fmean(step_ms), hbm, tfl)
        t_roof = max(bwork["bytes"] / (hbm * 1e9), bwork["flops"] / (tfl * 1e12)) * 1e3
        blk_roof.update({"t_roof_ms": round(t_roof, 4), "frac_time": round(t_roof / statistics.fmean(step_ms), 4),
                         "definition": "headline: masker read of x + idx + halo gather + residual + y + weights; "
                                       "halo-method FLOPs (SURVEY 8(d))"})
        if sched == L.SCHED_FUSED:
            bf = stats["block_fused"]
            t_f = max(bf["bytes"] / (hbm * 1e9), bf["flops"] / (tfl * 1e12)) * 1e3
            blk_roof["schedule_roofline"] = {
                "t_roof_ms": round(t_f, 4), "frac_time": round(t_f / statistics.fmean(step_ms), 4),
                "definition": "masker-fused schedule minimum: x once + h1 write + h1 halo reads + residual + y + "
                              "weights; dense-conv1 FLOPs"}
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(tot_max / K, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME if (h, c_in, c_mid) == (28, 512, 128) else
                       f"experiment: identity dyn-block {h}x{w}x{c_in} c_mid={c_mid}", "global_batch": world * n,
                       "per_gpu_batch": n,
                       "H": h, "W": w, "c_in": c_in, "c_mid": c_mid, "S": s, "r_target": wl["r"],
                       "r_patch": round(stats["r_patch"], 4), "r_pixel": round(stats["r_pixel"], 4),
                       "parallelism": f"dp{world}", "l2": "flushed (256 MiB read) before every timed step",
                       "launch": "CUDA graph replay" if args.graph else "eager (one launch per kernel, PDL)",
                       "schedule": sched_name},
            "latency_ms": {"p10": round(float(np.percentile(step_ms, 10)), 4),
                           "p50": round(float(np.percentile(step_ms, 50)), 4),
                           "p90": round(float(np.percentile(step_ms, 90)), 4)},
            "kernels_ms": {k2: round(v, 4) for k2, v in kern_ms.items()},
            "dense_ms_per_step": round(dense_max, 4),
            "speedup_vs_dense": round(dense_max / (tot_max / K), 3),
            "roofline": roof,
            "kernels_roofline": kern_roof,
            "network": net_info,
            "block_roofline": blk_roof,
            "e2e": {"value": round(e2e_val, 1), "unit": "images/s", "h2d_bytes_per_step": x.numel() * 2,
                    "d2h_bytes_per_step": x.numel() * 2,
                    "api": "DynBlock.stream_host: pinned host batches, H2D / compute / D2H on three streams, "
                           "consecutive steps overlapped; CUDA events around all K steps, L2 flushed before each",
                    "serial_value": round(ldist.throughput(n, world, K, e2e_serial_max), 1),
                    "serial_api": "DynBlock.forward_host: H2D, block, D2H back to back per step"},
            "stats": {"active_cells_all_ranks": int(act_all), "cells_all_ranks": int(cells_all),
                      "r_patch_all_ranks": round(act_all / max(cells_all, 1), 4),
                      "rank_ms_per_step": {"min": round(min(rank_ms), 4), "max": round(max(rank_ms), 4),
                                           "mean": round(statistics.fmean(rank_ms), 4)}},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(x_cpu, wts_cpu, wm_cpu, blk.bm, s, args.cpu_budget, n)
        if args.detail:
            with open(args.detail, "w") as f:
                json.dump({"line": line, "step_ms": step_ms, "dense_ms": dense_ms, "work": kwork,
                           "block": bwork, "dense": dwork, "stats": stats}, f, indent=1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def network_measure(world: int, steps: int, r: float = 0.5):
    """LAS-ResNet-101 forward (configs[2]): global batch 256 split over the ranks,
    224x224, S_net 4-4-2-1, masker biases calibrated to r on the activations each
    block sees; the forward and the dense-identity-block comparator each one CUDA
    graph.  Returns per-rank (ms_dyn, ms_dense, n_local, mean r_patch)."""
    import synth
    import paper_2210_06223_b200 as L

    n_local = max(1, 256 // world)
    wts = synth.make_lasnet_weights(seed=11)
    x = synth.make_image_batch(n_local, 224, seed=int(os.environ.get("RANK", "0"))).cuda()
    net = L.LASResNet(n_local, wts, hw=224, r=r)
    net.forward(x, calibrate_r=r)
    torch.cuda.synchronize()
    rate = statistics.fmean(float(b.mask_buf.float().mean().item()) for b in net.blocks())
    out = []
    for dense in (False, True):
        g = net.capture(x, dense=dense)
        for _ in range(2):
            g.replay()
        st = torch.cuda.current_stream()
        ev = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.replay()
            b.record(st)
            ev.append((a, b))
        torch.cuda.synchronize()
        out.append(statistics.median(a.elapsed_time(b) for a, b in ev))
        del g
    del net
    torch.cuda.empty_cache()
    return out[0], out[1], n_local, rate


def ctypes_array(events):
    import ctypes

    arr = (ctypes.c_void_p * len(events))()
    for i, e in enumerate(events):
        arr[i] = e.cuda_event
    return arr


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_lasnet(args)


if __name__ == "__main__":
    main()
