#!/usr/bin/env python
"""bench.py -- LASNet on B200: LAS-ResNet-101 images/s and dyn-block latency vs r / S.

Headline (BASELINE.json metric, configs[2]): the LAS-ResNet-101 forward at
ImageNet 224x224, global batch 256 sharded over the ranks (strong scaling),
S_net 4-4-2-1, masker biases calibrated on a separate batch so ~r = 0.5 of the
cells of every dynamic block are active, bf16, random-init weights, synthetic
N(0,1) images.  A step = one forward of the whole network on the rank's images
(stem -> pool -> 4 stages of blocks, each running masker -> compaction ->
gather+conv1 -> conv2 -> conv3+scatter-add -> head), one CUDA graph replay, plus
(N > 1) the all-gather of the logits over NCCL (SURVEY 8(e) exchange step).

Second half of the metric ("dyn-block latency vs activation rate"): the
configs[1] block (ResNet-50 stage-3 identity block, N = 128 per GPU, 28x28x512,
c_mid 128) at S = 4, r = 0.5 in full detail (`block`), and the grid
S in {1,2,4,7} x r in {0.25,0.5,0.75,1.0} (`block_sweep`).

Timing: W warm-up steps, then exactly K timed steps bracketed by barrier +
synchronize; CUDA events on the launching stream around every step (and one
pair around all K: `ms_per_step` = that pair / K).  Network: every input is
larger than L2 (image batch 213 MB, stage-1 maps 411 MB), no flush.  Block:
L2 flushed before every step by reading 256 MiB.  Max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lasnet|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N processes (one per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import ctypes
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
NET_BATCH = 256
NET_HW = 224
NET_R = 0.5
NET_WORKLOAD = ("LAS-ResNet-101 forward (BASELINE configs[2]): ImageNet 224x224, global batch 256 sharded over "
                "the GPUs, S_net 4-4-2-1, r = 0.5 (masker biases calibrated on a separate batch)")
WORKLOAD = dict(n=128, h=28, w=28, c_in=512, c_mid=128, s=4, r=0.5)
WORKLOAD_NAME = "resnet50-stage3 identity dyn-block (BASELINE configs[1]) N=128/GPU 28x28x512 c_mid=128 S=4 r=0.5"
SWEEP_S = (1, 2, 4, 7)
SWEEP_R = (0.25, 0.5, 0.75, 1.0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="lasnet", choices=["lasnet", "reference"])
    ap.add_argument("--s", type=int, default=WORKLOAD["s"], help="block sub-object: granularity S")
    ap.add_argument("--r", type=float, default=WORKLOAD["r"], help="block sub-object: activation rate")
    ap.add_argument("--n", type=int, default=WORKLOAD["n"], help="block sub-object: images per GPU")
    ap.add_argument("--hw", type=int, default=WORKLOAD["h"], help="(experiments) spatial size of the block")
    ap.add_argument("--c-in", type=int, default=WORKLOAD["c_in"], help="(experiments) block width")
    ap.add_argument("--c-mid", type=int, default=WORKLOAD["c_mid"], help="(experiments) bottleneck width")
    ap.add_argument("--net-r", type=float, default=NET_R, help="network activation rate target")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work per cpu_baseline")
    ap.add_argument("--no-sweep", action="store_true", help="skip the S x r block sweep")
    ap.add_argument("--no-block", action="store_true", help="skip the block sub-object")
    ap.add_argument("--no-coco", action="store_true", help="skip the COCO backbone sub-object (configs[4])")
    ap.add_argument("--no-regnet", action="store_true", help="skip the LAS-RegNetY sub-object (configs[3])")
    ap.add_argument("--detail", default=None, help="write per-kernel detail JSON here")
    ap.add_argument("--schedule", default="auto", choices=["auto", "separate", "fused"],
                    help="block sub-object: separate = north-star branch (masker, then gather+conv1 on halos); "
                         "fused = the paper's Table-1 schedule; auto = lasnet_choose_schedule(r)")
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
# Compulsory bytes and FLOPs of every kernel the library launches (DESIGN.md
# "Roofline accounting"; SURVEY 8(d) per-unit figures).  Bytes: each input read
# once and each output written once (h1 halo windows read once per active patch);
# FLOPs: 2 * MAC of the method's work (active output pixels, clipped halos).

def mask_geometry(mask_cells: np.ndarray, h, w, s, stride=1):
    """Active patches P, in-image halo pixels of their conv1 windows (at the input
    resolution: side stride*(S-1)+3, origin stride*S*g - 1), in-image output pixels."""
    n, gh, gw = mask_cells.shape
    ids = np.flatnonzero(mask_cells.reshape(-1))
    P = len(ids)
    g = ids % (gh * gw)
    gy, gx = g // gw, g % gw
    hi, wi, si = h * stride, w * stride, s * stride
    side = stride * (s - 1) + 3
    y0, x0 = gy * si - 1, gx * si - 1
    hy = np.minimum(y0 + side, hi) - np.maximum(y0, 0)
    hx = np.minimum(x0 + side, wi) - np.maximum(x0, 0)
    oy = np.minimum(gy * s + s, h) - gy * s
    ox = np.minimum(gx * s + s, w) - gx * s
    return dict(P=P, halo_px=int(np.sum(hy * hx)), out_px=int(np.sum(oy * ox)), side=side, cells=n * gh * gw)


def kernel_work(name: str, m: dict) -> dict:
    """bytes / flops of one launch of kernel `name` in the layer described by m:
    n, h, w (output), c_in, c_mid, c_out, stride, s, and for dynamic layers the
    mask geometry (P, halo_px, out_px, side, cells)."""
    e = 2
    n, h, w = m["n"], m.get("h", 0), m.get("w", 0)
    c_in, c_mid, c_out, st = m.get("c_in", 0), m.get("c_mid", 0), m.get("c_out", 0), m.get("stride", 1)
    px, pxi = n * h * w, n * h * w * st * st
    W1, W2, W3 = c_mid * c_in * e, 9 * c_mid * c_mid * e, c_out * c_mid * e
    P, halo, out, side = m.get("P", 0), m.get("halo_px", 0), m.get("out_px", 0), m.get("side", 0)
    ss, cells = m.get("s", 1) ** 2, m.get("cells", 0)
    win = P * side * side * c_mid * e
    k = {
        "stem_pack": (2 * 64 * 7 * 7 * 8 * e, 0),
        "stem_conv": (n * 2 * h * (2 * w + 8) * 8 * e + px * 64 * e + 64 * 448 * e, 2 * px * 64 * 147),
        "maxpool": (n * 4 * h * w * m.get("c", 0) * e + px * m.get("c", 0) * e, 0),
        "head": (n * m.get("hw", 0) * m.get("c", 0) * e + m.get("classes", 0) * m.get("c", 0) * e
                 + n * m.get("classes", 0) * 4, 2 * n * m.get("c", 0) * (m.get("hw", 0) + m.get("classes", 0))),
        "conv1_dense": (pxi * (c_in + c_mid) * e + W1, 2 * pxi * c_in * c_mid),
        "conv2_dense": (pxi * c_mid * e + px * c_mid * e + W2, 2 * px * 9 * c_mid * c_mid),
        "subsample": (2 * px * c_in * e, 0),
        # the dynamic projection block's dense shortcut R = Wd x_s + bd (masked ReLU epilogue)
        "shortcut": (px * c_in * e + px * c_out * e + c_out * c_in * e + cells, 2 * px * c_in * c_out),
        "add_bias": (3 * c_out * 4, 0),
        "conv23_dense": (px * c_mid * e + 2 * px * c_out * e + W2 + W3,
                         2 * px * (9 * c_mid * c_mid + c_mid * c_out)),
        "mask": (pxi * c_in * e + cells, 2 * pxi * c_in),
        "mask_compact": (pxi * c_in * e + cells + 4 * P, 2 * pxi * c_in),
        "compact": (cells + 4 * P, 0),
        "conv1_mask": (px * (c_in + c_mid) * e + px * 16 + W1, 2 * px * c_in * (c_mid + 1)),
        "decide": (px * 16 + cells + 4 * P, 0),
        "decide+ids": (px * 16 + cells + 4 * P, 0),
        "decide+gather": (px * 16 + cells + 4 * P + halo * c_mid * e + win, 0),
        "conv1_dyn": (halo * c_in * e + win + W1, 2 * halo * c_in * c_mid),
        "conv2_dyn": (win + P * ss * c_mid * e + W2, 2 * out * 9 * c_mid * c_mid),
        # conv2 gathering its im2col rows from the dense h1: the windows' in-image pixels once, h2 out
        "conv2_gather": (halo * c_mid * e + P * ss * c_mid * e + W2, 2 * out * 9 * c_mid * c_mid),
        "conv3_dyn": (P * ss * c_mid * e + 2 * out * c_out * e + W3, 2 * out * c_mid * c_out),
        "conv23": (win + 2 * out * c_out * e + W2 + W3, 2 * out * (9 * c_mid * c_mid + c_mid * c_out)),
        "conv23_direct": (halo * c_mid * e + 2 * out * c_out * e + W2 + W3,
                          2 * out * (9 * c_mid * c_mid + c_mid * c_out)),
    }
    if name == "conv3_dense":
        if m.get("proj"):  # [h2 | x_s] x [W3 | Wd]^T, no residual read
            b, f = px * (c_mid + c_in) * e + px * c_out * e + c_out * (c_mid + c_in) * e, 2 * px * (c_mid + c_in) * c_out
        else:
            b, f = px * c_mid * e + 2 * px * c_out * e + W3, 2 * px * c_mid * c_out
        return {"bytes": int(b), "flops": int(f)}
    if name not in k:
        return {"bytes": 0, "flops": 0}
    b, f = k[name]
    return {"bytes": int(b), "flops": int(f)}


def algorithmic_work(mask_cells: np.ndarray, n, h, w, c_in, c_mid, c_out, s):
    """The configs[1] block: per-kernel work of both schedules, the SURVEY 8(d)
    headline block work, the dense block, and mask statistics."""
    g = mask_geometry(mask_cells, h, w, s)
    m = dict(n=n, h=h, w=w, c_in=c_in, c_mid=c_mid, c_out=c_out, s=s, **g)
    names = ["mask_compact", "conv1_dyn", "conv23", "conv2_dyn", "conv3_dyn", "conv1_mask", "decide+ids", "decide",
             "decide+gather", "conv23_direct"]
    k = {nm: kernel_work(nm, m) for nm in names}
    e = 2
    W = (c_mid * c_in + 9 * c_mid * c_mid + c_out * c_mid) * e
    P, halo, out = g["P"], g["halo_px"], g["out_px"]
    block = dict(bytes=n * h * w * c_in * e + g["cells"] + 4 * P + halo * c_in * e + 2 * out * c_out * e + W,
                 flops=k["conv1_dyn"]["flops"] + k["conv2_dyn"]["flops"] + k["conv3_dyn"]["flops"])
    block_fused = dict(bytes=n * h * w * (c_in + c_mid) * e + g["cells"] + 4 * P + halo * c_mid * e
                       + 2 * out * c_out * e + W,
                       flops=2 * n * h * w * c_in * c_mid + k["conv2_dyn"]["flops"] + k["conv3_dyn"]["flops"])
    dense = dict(bytes=2 * n * h * w * c_in * e + W,
                 flops=2 * n * h * w * (c_in * c_mid + 9 * c_mid * c_mid + c_mid * c_out))
    return k, block, dense, dict(P=P, halo_px=halo, out_px=out, r_patch=P / max(g["cells"], 1),
                                 r_pixel=out / (n * h * w), block_fused=block_fused)


def roofline_entry(work, ms, hbm, tfl):
    t_hbm = work["bytes"] / (hbm * 1e9)
    t_tc = work["flops"] / (tfl * 1e12)
    if t_hbm >= t_tc:
        ach = work["bytes"] / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4)}
    ach = work["flops"] / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": tfl, "unit": "TFLOP/s", "frac": round(ach / tfl, 4)}


def t_roof_ms(work, hbm, tfl):
    return max(work["bytes"] / (hbm * 1e9), work["flops"] / (tfl * 1e12)) * 1e3


def ncu_traffic(kernel: str, scope: str = "net"):
    """DRAM bytes (read + write) per launch of `kernel` from the latest committed ncu
    evidence (profiles/ncu_full_<tag>.json), or (None, None).  scope "net": the mean
    over that kernel's launches in one eager LAS-R101 forward (r2 layout); "block":
    the --set full capture of the configs[1] block (conv23_direct is the conv23
    kernel reading the dense h1)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_*.json")))
    for f in reversed(files):
        d = json.load(open(f))
        if scope == "net" and isinstance(d.get("net"), list):
            for e in d["net"]:
                if e.get("kernel") == kernel:
                    return int(e.get("dram_read", 0) + e.get("dram_write", 0)), os.path.relpath(f, ROOT)
        if scope == "block":
            want = "conv23" if kernel.startswith("conv23") else kernel
            for e in d.get("full", []):
                if e.get("capture", "block") == "block" and e.get("kernel") in (want, kernel) and "launches" not in e:
                    return int(e.get("dram_read", 0) + e.get("dram_write", 0)), os.path.relpath(f, ROOT)
    return None, None


def ctypes_array(events):
    arr = (ctypes.c_void_p * len(events))()
    for i, e in enumerate(events):
        arr[i] = e.cuda_event
    return arr


def ev_pair():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


# ------------------------------------------------------------ cpu oracle ----

def oracle_block_sample(x_cpu, wts_cpu, wm_cpu, bm, s, k_images, threads):
    """The oracle as it stands on the first k images: masker -> compact -> literal
    gather/conv/scatter block.  Returns seconds."""
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


def cpu_baseline_block(x_cpu, wts_cpu, wm_cpu, bm, s, budget_s, n_total):
    import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    t1 = oracle_block_sample(x_cpu, wts_cpu, wm_cpu, bm, s, 2, threads)
    k = int(max(2, min(n_total, budget_s / max(t1 / 2, 1e-6))))
    t = oracle_block_sample(x_cpu, wts_cpu, wm_cpu, bm, s, k, threads) if k > 2 else t1
    return {"value": round(k / t, 2), "unit": "images/s", "cores": threads, "kind": "oracle",
            "sample": f"first {k} of the {n_total} images, same S/weights/masker bias, fp64 literal mode "
                      f"(masker+compact+gather/conv/scatter), OpenMP over patches; {t:.2f} s"}


def oracle_net_sample(x_img, weights, net_meta, k_images, threads):
    """The oracle LAS-ResNet-101 forward (oracle.lasnet_forward, fp64, the GPU
    network's masker biases) on the first k images.  Returns seconds."""
    import oracle
    import synth

    oracle.set_threads(threads)
    xd = synth.to_f64(x_img[:k_images])[:, :, 4:4 + x_img.shape[1], :]
    t0 = time.perf_counter()
    oracle.lasnet_forward(xd, synth.weights_f64_nested(weights), net_meta)
    return time.perf_counter() - t0


def cpu_baseline_net(x_img, weights, net_meta, budget_s):
    import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    t1 = oracle_net_sample(x_img, weights, net_meta, 1, threads)
    k = int(max(1, min(x_img.shape[0], budget_s / max(t1, 1e-6))))
    t = oracle_net_sample(x_img, weights, net_meta, k, threads) if k > 1 else t1
    return {"value": round(k / t, 3), "unit": "images/s", "cores": threads, "kind": "oracle",
            "sample": f"{k} of the {x_img.shape[0]} images of the rank's batch through oracle.lasnet_forward (fp64: "
                      f"stem, pool, every block with the GPU network's masker biases -- masker, compaction, literal "
                      f"gather/conv/scatter -- head); {t:.2f} s on {threads} host threads"}


# ------------------------------------------------------------- reference ----

def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (this tier's
    reference arm; the paper ships no code), timed on the lasnet arm's workload
    (the LAS-ResNet-101 forward), each step a bounded sample of the batch."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth

    oracle.build()
    world = max(1, args.gpus)
    n_loc = NET_BATCH // world
    weights = synth.make_lasnet_weights(seed=11)
    x = synth.make_image_batch(n_loc, NET_HW, seed=0)
    meta = synth.lasnet_oracle_biases(weights, seed=5000)
    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    # the oracle calibrates its masker biases on a separate image (untimed), like the GPU arm
    xc = synth.make_image_batch(1, NET_HW, seed=5000)
    oracle.lasnet_forward(synth.to_f64(xc)[:, :, 4:4 + NET_HW, :], synth.weights_f64_nested(weights), meta,
                          calibrate_r=NET_R)
    t1 = oracle_net_sample(x, weights, meta, 1, threads)
    k_img = int(max(1, min(n_loc, 3.0 / max(t1, 1e-6))))
    for _ in range(args.warmup):
        oracle_net_sample(x, weights, meta, k_img, threads)
    ts = [oracle_net_sample(x, weights, meta, k_img, threads) for _ in range(args.steps)]
    tot = sum(ts)
    val = k_img * args.steps / tot
    line = {"metric": METRIC, "value": round(val, 4), "unit": "images/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": NET_WORKLOAD, "global_batch": NET_BATCH, "sample_images_per_step": k_img,
                       "r_target": NET_R, "s_net": "4-4-2-1"},
            "cpu_baseline": {"value": round(val, 4), "unit": "images/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {k_img} of the rank's {n_loc} images per step, oracle.lasnet_forward "
                                       f"(masker biases from a fixed-seed oracle calibration)"},
            "e2e": {"value": round(val, 4), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- network ----

def net_layer_meta(t: dict) -> dict:
    """Layer description of one traced LASResNet call (for kernel_work)."""
    kind, o = t["kind"], t["obj"]
    if kind in ("stem", "maxpool", "head"):
        return {k: v for k, v in t.items() if k not in ("kind", "obj", "ev0", "ev1")}
    if kind == "proj":
        d = o.desc
        m = dict(n=d.n, h=d.h, w=d.w, c_in=d.c_in, c_mid=d.c_mid, c_out=d.c_out, stride=d.stride, s=d.s, proj=True)
        if getattr(o, "dynamic", False):
            m.update(mask_geometry(o.mask_buf.cpu().numpy(), d.h, d.w, d.s, d.stride), proj=False, shortcut=True)
        return m
    sh = o.shape
    m = dict(n=sh.n, h=sh.h, w=sh.w, c_in=sh.c_in, c_mid=sh.c_mid, c_out=o.c_out, stride=1, s=sh.s)
    if kind == "dyn":
        m.update(mask_geometry(o.mask_buf.cpu().numpy(), sh.h, sh.w, sh.s))
    return m


def net_block_literal_work(t: dict, hbm, tfl):
    """SURVEY 8(d) headline (north-star literal) definition of one dynamic layer."""
    m = net_layer_meta(t)
    e = 2
    st = m.get("stride", 1)
    W = (m["c_mid"] * m["c_in"] + 9 * m["c_mid"] ** 2 + m["c_out"] * m["c_mid"]) * e
    px_in = m["n"] * m["h"] * m["w"] * st * st
    b = px_in * m["c_in"] * e + m["cells"] + 4 * m["P"] + m["halo_px"] * m["c_in"] * e + 2 * m["out_px"] * m["c_out"] * e + W
    f = 2 * (m["halo_px"] * m["c_in"] * m["c_mid"] + m["out_px"] * 9 * m["c_mid"] ** 2 + m["out_px"] * m["c_mid"] * m["c_out"])
    if m.get("shortcut"):  # dense projection shortcut of a dynamic first block
        px = m["n"] * m["h"] * m["w"]
        b += px * m["c_in"] * e + px * m["c_out"] * e + m["c_out"] * m["c_in"] * e
        f += 2 * px * m["c_in"] * m["c_out"]
    return {"bytes": b, "flops": f}


def network_measure(args, world, rank, local, hbm, tfl):
    """The headline: LAS-ResNet-101 forward on this rank's shard of the global batch."""
    import torch.distributed as dist

    import synth
    import paper_2210_06223_b200 as L
    from paper_2210_06223_b200 import _lib, dist as ldist

    lib = _lib.load()
    lo, hi = ldist.shard(NET_BATCH, rank, world)
    n_loc = hi - lo
    weights = synth.make_lasnet_weights(seed=11)
    x_cpu = synth.make_image_batch(n_loc, NET_HW, seed=100 + rank)
    net = L.LASResNet(n_loc, weights, hw=NET_HW, r=args.net_r)
    # masker biases calibrated on a separate batch of the same distribution
    net.forward(synth.make_image_batch(n_loc, NET_HW, seed=5000 + rank).cuda(), calibrate_r=args.net_r)
    x = x_cpu.cuda()
    stream = torch.cuda.current_stream()

    # eager forward with an event pair around every kernel: names, per-launch times, work
    nmax = 512
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nmax)]
    for e in evs:
        e.record(stream)
    handles = ctypes_array(evs)
    trace_ms = []
    for rep in range(3):
        trace = []
        lib.lasnet_set_kernel_events(handles, nmax)
        net.forward(x, trace=trace)
        nev = int(lib.lasnet_kernel_event_count())
        names = [lib.lasnet_kernel_event_name(i).decode() for i in range(nev)]
        lib.lasnet_set_kernel_events(None, 0)
        torch.cuda.synchronize()
        trace_ms.append([evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(nev)])
    launches_per_step = net.launches
    kms = [statistics.median(v) for v in zip(*trace_ms[1:])]
    launches = []  # (name, layer kind, stage, ms, work)
    for t in trace:
        m = net_layer_meta(t)
        for i in range(t["ev0"], t["ev1"]):
            launches.append(dict(name=names[i], kind=t["kind"], stage=t.get("stage"), ms=kms[i],
                                 work=kernel_work(names[i], m)))
    # per-stage dynamic activation statistics (SURVEY 8(e) exchange step below)
    act = [int(b.count.item()) for b in net.blocks()]
    cells = [b.ncells for b in net.blocks()]

    # headline: the forward as one CUDA graph; N > 1 adds the logits all-gather (NCCL)
    g = net.capture(x)
    gathered = torch.empty((n_loc * world, net.logits.shape[1]), dtype=torch.float32, device="cuda")

    def step():
        g.replay()
        if world > 1:
            ldist.exchange_logits(net.logits, gathered)

    for _ in range(max(args.warmup, 3)):
        step()
    K = args.steps
    ev = [ev_pair() for _ in range(K)]
    tot = ev_pair()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tot[0].record(stream)
    for k in range(K):
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    tot[1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = tot[0].elapsed_time(tot[1])
    logits = net.logits.clone()
    del g

    # dense comparator: the same network with the identity blocks run on every pixel
    gd = net.capture(x, dense=True)
    for _ in range(3):
        gd.replay()
    td = ev_pair()
    torch.cuda.synchronize()
    td[0].record(stream)
    for _ in range(K):
        gd.replay()
    td[1].record(stream)
    torch.cuda.synchronize()
    dense_ms = td[0].elapsed_time(td[1]) / K
    del gd

    # end to end through the public API: pinned host images -> logits on the host
    x_host = x_cpu.pin_memory()
    lg_host = [torch.empty_like(net.logits, device="cpu").pin_memory() for _ in range(2)]
    x_devs = [x, torch.empty_like(x)]
    graphs = [net.capture(xd) for xd in x_devs]
    net.stream_host([x_host], lg_host, x_devs, graphs, 2)
    torch.cuda.synchronize()
    te = ev_pair()
    te[0].record(stream)
    net.stream_host([x_host], lg_host, x_devs, graphs, K)
    te[1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = te[0].elapsed_time(te[1])
    assert torch.equal(lg_host[(K - 1) % 2], logits.cpu()), "e2e logits differ from the device-timed forward"
    del graphs

    tot_max, dense_max, e2e_max = ldist.max_over_ranks([tot_ms, dense_ms, e2e_ms], device="cuda")
    act_all = ldist.active_counts(act + cells, device="cuda")
    rank_ms = ldist.gather_over_ranks(tot_ms / K, device="cuda")
    res = dict(n_loc=n_loc, step_ms=step_ms, tot_ms=tot_ms, tot_max=tot_max, dense_ms=dense_max, e2e_ms=e2e_max,
               launches=launches, trace=trace, launches_per_step=launches_per_step, rank_ms=rank_ms,
               act_all=act_all[:len(act)], cells_all=act_all[len(act):], x_cpu=x_cpu, weights=weights, net=net,
               h2d=x_cpu.numel() * 2, d2h=net.logits.numel() * 4)
    return res


def summarize_network(res, world, hbm, tfl, args):
    """JSON pieces of the headline from network_measure's raw results (rank 0)."""
    K = args.steps
    launches = res["launches"]
    # kernels grouped by name: the dominant one (largest share of the eager forward)
    groups = {}
    for l in launches:
        gk = groups.setdefault(l["name"], {"ms": 0.0, "bytes": 0, "flops": 0, "launches": 0})
        gk["ms"] += l["ms"]
        gk["bytes"] += l["work"]["bytes"]
        gk["flops"] += l["work"]["flops"]
        gk["launches"] += 1
    eager_ms = sum(l["ms"] for l in launches)
    dom = max(groups, key=lambda k: groups[k]["ms"])
    gd = groups[dom]
    roof = roofline_entry(gd, gd["ms"], hbm, tfl)
    traffic, tsrc = ncu_traffic(dom)
    roof.update({"kernel": dom, "launches_per_forward": gd["launches"],
                 "traffic": traffic, "traffic_source": tsrc,
                 "algorithmic_per_launch": {"bytes": gd["bytes"] // gd["launches"],
                                            "flops": gd["flops"] // gd["launches"]},
                 "avg_launch_ms": round(gd["ms"] / gd["launches"], 5),
                 "share_of_forward": round(gd["ms"] / eager_ms, 3),
                 "timing": "CUDA events around every launch of this kernel in an eager forward (median of 2), "
                           "summed; achieved = summed algorithmic bytes (or FLOPs) / summed time"})
    kern_table = {}
    for k, v in sorted(groups.items(), key=lambda kv: -kv[1]["ms"]):
        e = roofline_entry(v, v["ms"], hbm, tfl)
        kern_table[k] = {"ms": round(v["ms"], 4), "launches": v["launches"], "share": round(v["ms"] / eager_ms, 3),
                         "bound": e["bound"], "frac": e["frac"]}
    # network rooflines: sum over launches of the per-kernel bound (what the schedule moves)
    # and, for the dynamic layers, the SURVEY 8(d) literal definition
    t_sched = sum(t_roof_ms(l["work"], hbm, tfl) for l in launches)
    t_lit = 0.0
    for t in res["trace"]:
        if t["kind"] == "dyn" or (t["kind"] == "proj" and getattr(t["obj"], "dynamic", False)):
            t_lit += t_roof_ms(net_block_literal_work(t, hbm, tfl), hbm, tfl)
        else:
            for i in range(t["ev0"], t["ev1"]):
                t_lit += t_roof_ms(launches[i]["work"], hbm, tfl)
    ms = res["tot_max"] / K
    per_stage = {}
    for l in launches:
        key = f"stage{l['stage']}_{l['kind']}" if l["stage"] is not None else l["kind"]
        per_stage[key] = round(per_stage.get(key, 0.0) + l["ms"], 4)
    return dict(ms=ms, roof=roof, kern_table=kern_table, t_sched=t_sched, t_lit=t_lit, eager_ms=eager_ms,
                per_stage=per_stage)


# ------------------------------------------------------------------ block ----

def block_measure(args, world, rank, hbm, tfl):
    """configs[1] block at (S, r) in full detail (latency, kernels, rooflines, dense,
    e2e); returns a dict (rank-local values; caller reduces)."""
    import synth
    import paper_2210_06223_b200 as L
    from paper_2210_06223_b200 import _lib

    lib = _lib.load()
    n, h, w, c_in, c_mid, s, r = args.n, args.hw, args.hw, args.c_in, args.c_mid, args.s, args.r
    x_cpu = synth.make_x(n, h, w, c_in, seed=0 + 7919 * rank)
    wts_cpu = synth.make_block_weights(c_in, c_mid, c_in, seed=1)
    wm_cpu = synth.make_masker_weights(c_in, seed=2)
    if args.schedule == "auto":
        sched = L.choose_schedule(n, h, w, c_in, c_mid, c_in, s, r)
    else:
        sched = L.SCHED_FUSED if args.schedule == "fused" else L.SCHED_SEPARATE
    blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts_cpu, wm_cpu, 0.0,
                     schedule=L.SCHED_FUSED if sched == L.SCHED_FUSED else None)
    blk.calibrate_bias(synth.make_x(n, h, w, c_in, seed=1000 + rank).cuda(), r)
    x = x_cpu.cuda()
    y = torch.empty_like(x)
    y2 = torch.empty_like(x)
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")  # 256 MiB read > 126 MB L2
    stream = torch.cuda.current_stream()

    def prep():
        y.copy_(x)
        flush.sum()

    for _ in range(max(args.warmup, 3)):
        prep()
        blk.forward(y)
    torch.cuda.synchronize()
    mask_cells = blk.mask_buf.cpu().numpy()
    kwork, bwork, dwork, stats = algorithmic_work(mask_cells, n, h, w, c_in, c_mid, c_in, s)
    K = args.steps
    l0 = blk.launches
    prep()
    blk.forward(y)
    n_launch = blk.launches - l0
    graph = blk.capture(y)
    for _ in range(2):
        prep()
        graph.replay()
    ev = [ev_pair() for _ in range(K)]
    torch.cuda.synchronize()
    for k in range(K):
        prep()
        ev[k][0].record(stream)
        graph.replay()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # breakdown pass: events around every kernel (named by the library)
    nk = 8
    evk = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nk)] for _ in range(K)]
    for row in evk:
        for e in row:
            e.record(stream)
    handles = [ctypes_array(row) for row in evk]
    names = None
    for k in range(K):
        prep()
        lib.lasnet_set_kernel_events(handles[k], nk)
        blk.forward(y)
        cnt = int(lib.lasnet_kernel_event_count())
        names = [lib.lasnet_kernel_event_name(i).decode() for i in range(cnt)]
    lib.lasnet_set_kernel_events(None, 0)
    torch.cuda.synchronize()
    kern_ms = {nm: statistics.fmean(evk[k][2 * i].elapsed_time(evk[k][2 * i + 1]) for k in range(K))
               for i, nm in enumerate(names)}
    # dense comparator
    for _ in range(3):
        flush.sum()
        blk.dense(x, y2)
    dms = []
    for k in range(K):
        flush.sum()
        a, b = ev_pair()
        a.record(stream)
        blk.dense(x, y2)
        b.record(stream)
        dms.append((a, b))
    torch.cuda.synchronize()
    dense_ms = statistics.fmean(a.elapsed_time(b) for a, b in dms)
    # e2e: pinned host batches through DynBlock.stream_host (H2D / block / D2H overlapped)
    x_host = x_cpu.pin_memory()
    y_host = [torch.empty_like(x_cpu).pin_memory() for _ in range(2)]
    y_b = torch.empty_like(y)
    blk.stream_host([x_host], y_host, [y, y_b], 2)
    torch.cuda.synchronize()
    a, b = ev_pair()
    a.record(stream)
    blk.stream_host([x_host], y_host, [y, y_b], K, before_step=lambda i: flush.sum())
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b)
    return dict(blk=blk, sched=sched, step_ms=step_ms, kern_ms=kern_ms, kwork=kwork, bwork=bwork, stats=stats,
                dense_ms=dense_ms, e2e_ms=e2e_ms, n_launch=n_launch, x_cpu=x_cpu, wts_cpu=wts_cpu, wm_cpu=wm_cpu,
                bytes_io=x.numel() * 2)


def block_sweep(args, rank, hbm, tfl):
    """configs[1] block latency vs S x r (graph replays, L2 flushed before each)."""
    import synth
    import paper_2210_06223_b200 as L

    n, h, w, c_in, c_mid = args.n, args.hw, args.hw, args.c_in, args.c_mid
    x = synth.make_x(n, h, w, c_in, seed=0 + 7919 * rank).cuda()
    xc = synth.make_x(n, h, w, c_in, seed=1000 + rank).cuda()
    wts = synth.make_block_weights(c_in, c_mid, c_in, seed=1)
    wm = synth.make_masker_weights(c_in, seed=2)
    y = torch.empty_like(x)
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    steps = max(5, min(args.steps, 10))
    out = []
    dense_ms = None
    for s in SWEEP_S:
        for r in SWEEP_R:
            sched = L.choose_schedule(n, h, w, c_in, c_mid, c_in, s, r)
            blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts, wm, 0.0,
                             schedule=L.SCHED_FUSED if sched == L.SCHED_FUSED else None)
            blk.calibrate_bias(xc, r)
            y.copy_(x)
            blk.forward(y)
            torch.cuda.synchronize()
            mc = blk.mask_buf.cpu().numpy()
            g = blk.capture(y)
            ms = []
            for k in range(steps + 2):
                y.copy_(x)
                flush.sum()
                a, b = ev_pair()
                a.record(stream)
                g.replay()
                b.record(stream)
                if k >= 2:
                    ms.append((a, b))
            if dense_ms is None:
                y2 = torch.empty_like(x)
                dd = []
                for k in range(steps + 2):
                    flush.sum()
                    a, b = ev_pair()
                    a.record(stream)
                    blk.dense(x, y2)
                    b.record(stream)
                    if k >= 2:
                        dd.append((a, b))
                torch.cuda.synchronize()
                dense_ms = statistics.fmean(a.elapsed_time(b) for a, b in dd)
            torch.cuda.synchronize()
            t = statistics.fmean(a.elapsed_time(b) for a, b in ms)
            _, bwork, _, st = algorithmic_work(mc, n, h, w, c_in, c_mid, c_in, s)
            tr = t_roof_ms(bwork, hbm, tfl)
            out.append({"S": s, "r_target": r, "r_patch": round(st["r_patch"], 4), "ms": round(t, 4),
                        "schedule": "fused" if sched == L.SCHED_FUSED else "separate",
                        "speedup_vs_dense": round(dense_ms / t, 3), "roofline_frac": round(tr / t, 4)})
            del g, blk
    return {"points": out, "dense_ms": round(dense_ms, 4),
            "timing": f"mean of {steps} CUDA-graph replays per point, L2 flushed (256 MiB read) before each; "
                      "schedule from lasnet_choose_schedule(r); masker bias calibrated on a separate batch; "
                      "roofline_frac = SURVEY 8(d) headline T_roof / measured"}


# ----------------------------------------------------------- COCO backbone ----

def coco_measure(args, rank):
    """BASELINE configs[4]: the LAS-ResNet-101 backbone at COCO 800x1333 (padded to
    800x1344), 8 images per GPU, S_net 4-4-2-1 and 4-4-7-1, r = 0.5,
    detection-shaped stage outputs (200x336 ... 25x42); one CUDA graph per forward,
    the dense comparator the same backbone with every block static."""
    import synth
    import paper_2210_06223_b200 as L

    n, hw = 8, (800, 1344)
    weights = synth.make_lasnet_weights(seed=11)
    x = synth.make_image_batch(n, hw, seed=200 + rank).cuda()
    xc = synth.make_image_batch(n, hw, seed=6000 + rank).cuda()
    stream = torch.cuda.current_stream()
    steps = max(3, min(args.steps, 10))
    out = {}
    for s_net in ((4, 4, 2, 1), (4, 4, 7, 1)):
        net = L.LASResNet(n, weights, hw=hw, s_net=s_net, r=0.5, backbone=True)
        net.forward(xc, calibrate_r=0.5)
        res = {}
        for dense in (False, True):
            g = net.capture(x, dense=dense)
            for _ in range(2):
                g.replay()
            a, b = ev_pair()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(steps):
                g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            res[dense] = a.elapsed_time(b) / steps
            del g
        r_blocks = [int(b.count.item()) / b.ncells for b in net.blocks()]
        key = "s_net_" + "-".join(map(str, s_net))
        out[key] = {"ms_per_forward": round(res[False], 4), "images_per_s": round(n / (res[False] * 1e-3), 1),
                    "ms_per_image": round(res[False] / n, 4), "dense_ms_per_forward": round(res[True], 4),
                    "speedup_vs_dense": round(res[True] / res[False], 3),
                    "r_patch_mean": round(statistics.fmean(r_blocks), 4)}
        del net
        torch.cuda.empty_cache()
    out.update({"workload": "LAS-ResNet-101 backbone (BASELINE configs[4]): 8 images/GPU of 800x1344 (1333 padded "
                            "to a multiple of 32), stage outputs 200x336 / 100x168 / 50x84 / 25x42, r = 0.5",
                "timing": f"mean of {steps} CUDA-graph replays per forward", "paper_context_ms_per_image": {
                    "V100 4-4-2-1": 30.7, "V100 4-4-7-1": 25.3, "V100 static": 39.5, "note": "P:400-405, batch 1"}})
    return out


# ---------------------------------------------------------------- config 1 ----

def config1_measure(args):
    """BASELINE configs[0] / SURVEY C1: one block, N = 1, 14x14x256, c_mid 64, S = 2,
    fp32 (the CUDA-core path), 25 of 49 cells active (masker bias calibrated on the
    input itself, so exactly 25 cells pass); CUDA-graph replays, inputs L2-resident.
    Latency-bound by construction: its roofline is ~0.29 us (21.7 MFLOP at the fp32
    SIMT peak)."""
    import synth
    import paper_2210_06223_b200 as L

    n, h, w, c, cm, s = 1, 14, 14, 256, 64, 2
    x = synth.make_x(n, h, w, c, seed=0, dtype="f32").cuda()
    wts = synth.make_block_weights(c, cm, c, seed=1, dtype="f32")
    # one lasnet_block_forward call: the single-launch small-batch block (small_block.cu)
    blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s, torch.float32), wts, synth.make_masker_weights(c, seed=2), 0.0,
                     schedule=L.SCHED_SEPARATE)
    blk.calibrate_bias(x, 25 / 49)
    # the step-by-step calls (mask_compact, dyn_block: 4 launches), for reference
    steps_blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s, torch.float32), wts, synth.make_masker_weights(c, seed=2),
                           blk.bm)
    y, y2 = x.clone(), torch.empty_like(x)
    blk.forward(y)
    torch.cuda.synchronize()
    active = int(blk.count.item())
    g = blk.capture(y)
    stream = torch.cuda.current_stream()
    steps = 200

    def timed(fn):
        for _ in range(10):
            fn()
        a, b = ev_pair()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps * 1e3

    dyn_us = timed(g.replay)
    y3 = x.clone()
    steps_blk.forward(y3)
    torch.cuda.synchronize()
    gs = steps_blk.capture(y3)
    steps_us = timed(gs.replay)
    gd = torch.cuda.CUDAGraph()
    blk.dense(x, y2)
    torch.cuda.synchronize()
    with torch.cuda.graph(gd):
        blk.dense(x, y2)
    dense_us = timed(gd.replay)
    return {"workload": "BASELINE configs[0]: one bottleneck block, N=1, 14x14x256, c_mid 64, S=2, fp32 (CUDA cores)",
            "active_cells": active, "cells": 49, "us_per_block": round(dyn_us, 2), "dense_us": round(dense_us, 2),
            "launch": "one cooperative launch per block (masker, compaction, conv1 on the dilated union of the active "
                      "cells, conv2, conv3 + scatter-add; the dense comparator likewise)",
            "us_per_block_step_kernels": round(steps_us, 2),
            "speedup_vs_dense": round(dense_us / dyn_us, 3), "roofline_us": 0.29,
            "roofline_frac": round(0.29 / dyn_us, 4), "tolerance": "1e-5 max-abs-rel (fp32 path, tests)",
            "timing": f"{steps} CUDA-graph replays in one event pair, inputs L2-resident; latency-bound by "
                      "construction (dependent phases behind grid barriers)"}


# ------------------------------------------------------------ LAS-RegNetY ----

def regnet_measure(args, rank, world):
    """BASELINE configs[3]: LAS-RegNetY-800MF at ImageNet 224x224, global batch 512
    sharded over the ranks, S_net 4-4-2-1, r = 0.5 (masker biases calibrated on a
    separate batch); one CUDA graph per forward; the dense comparator runs every
    identity Y-block static."""
    import synth
    import paper_2210_06223_b200 as L
    from paper_2210_06223_b200 import dist as ldist

    lo, hi = ldist.shard(512, rank, world)
    n = hi - lo
    weights = synth.make_regnet_weights(seed=21)
    x = synth.make_image_batch(n, 224, seed=300 + rank).cuda()
    net = L.LASRegNet(n, weights, hw=224)
    net.forward(synth.make_image_batch(n, 224, seed=7000 + rank).cuda(), calibrate_r=0.5)
    stream = torch.cuda.current_stream()
    steps = max(3, min(args.steps, 10))
    res = {}
    for dense in (False, True):
        g = net.capture(x, dense=dense)
        for _ in range(2):
            g.replay()
        a, b = ev_pair()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(steps):
            g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        res[dense] = a.elapsed_time(b) / steps
        del g
    r_blocks = [int(b.count.item()) / b.ncells for b in net.blocks()]
    t_dyn, t_dense = ldist.max_over_ranks([res[False], res[True]], device="cuda")
    del net
    torch.cuda.empty_cache()
    return {"workload": "LAS-RegNetY-800MF forward (BASELINE configs[3]): 224x224, global batch 512 sharded over the "
                        "GPUs, S_net 4-4-2-1 (identity Y-blocks dynamic, stage-first blocks static), r = 0.5; widths "
                        "zero-padded to multiples of 64",
            "per_gpu_batch": n, "ms_per_forward": round(t_dyn, 4), "images_per_s": round(512 / (t_dyn * 1e-3), 1),
            "dense_ms_per_forward": round(t_dense, 4), "speedup_vs_dense": round(t_dense / t_dyn, 3),
            "r_patch_mean": round(statistics.fmean(r_blocks), 4),
            "timing": f"mean of {steps} CUDA-graph replays per forward, max over ranks"}


# ---------------------------------------------------------------- lasnet ----

def run_lasnet(args):
    import torch.distributed as dist

    from paper_2210_06223_b200 import _lib, build, dist as ldist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0 or not os.path.exists(_lib.LIB_PATH):
        build.build()
    if world > 1:
        dist.barrier()
    _lib.load()
    hbm, tfl, tfl_sus, psrc = peaks()

    sampler = ClockSampler(local)
    sampler.start()
    net = network_measure(args, world, rank, local, hbm, tfl)
    blk = None if args.no_block else block_measure(args, world, rank, hbm, tfl)
    sweep = None if args.no_sweep else block_sweep(args, rank, hbm, tfl)
    coco = None if args.no_coco else coco_measure(args, rank)
    regnet = None if args.no_regnet else regnet_measure(args, rank, world)
    c1 = None if args.no_block else config1_measure(args)
    clocks = sampler.stop()
    if blk is not None:
        b_tot = sum(blk["step_ms"])
        b_max, b_dense, b_e2e = ldist.max_over_ranks([b_tot, blk["dense_ms"], blk["e2e_ms"]], device="cuda")

    if rank == 0:
        K = args.steps
        sm = summarize_network(net, world, hbm, tfl, args)
        value = NET_BATCH / (sm["ms"] * 1e-3)
        e2e_val = NET_BATCH * K / (net["e2e_ms"] * 1e-3)
        r_blocks = [a / c for a, c in zip(net["act_all"], net["cells_all"])]
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(sm["ms"], 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": NET_WORKLOAD, "model": "LAS-ResNet-101", "global_batch": NET_BATCH,
                       "per_gpu_batch": net["n_loc"], "image": f"{NET_HW}x{NET_HW}", "s_net": "4-4-2-1",
                       "r_target": args.net_r, "r_patch_mean": round(statistics.fmean(r_blocks), 4),
                       "parallelism": f"dp{world}", "l2": "inputs larger than L2 (213 MB image batch, 411 MB "
                       "stage-1 maps); no flush", "launch": "one CUDA graph replay per forward"
                       + (" + NCCL all_gather_into_tensor of the logits" if world > 1 else "")},
            "latency_ms": {"p10": round(float(np.percentile(net["step_ms"], 10)), 4),
                           "p50": round(float(np.percentile(net["step_ms"], 50)), 4),
                           "p90": round(float(np.percentile(net["step_ms"], 90)), 4)},
            "dense_identity_ms_per_step": round(net["dense_ms"], 4),
            "speedup_vs_dense": round(net["dense_ms"] / sm["ms"], 3),
            "roofline": sm["roof"],
            "network_roofline": {
                "t_roof_schedule_ms": round(sm["t_sched"], 4), "frac_schedule": round(sm["t_sched"] / sm["ms"], 4),
                "t_roof_literal_ms": round(sm["t_lit"], 4), "frac_literal": round(sm["t_lit"] / sm["ms"], 4),
                "definition": "schedule: sum over every launch of max(algorithmic bytes / HBM peak, FLOPs / tensor "
                              "peak); literal: the dynamic layers by the SURVEY 8(d) headline definition (masker "
                              "read of x + idx + halo gather + residual + y + weights, halo-method FLOPs), the "
                              "static layers as launched", "peaks": {"hbm_gbs": hbm, "bf16_tflops": tfl,
                                                                       "source": psrc}},
            "kernels": sm["kern_table"],
            "eager_breakdown_ms": sm["per_stage"],
            "e2e": {"value": round(e2e_val, 1), "unit": "images/s", "h2d_bytes_per_step": net["h2d"],
                    "d2h_bytes_per_step": net["d2h"],
                    "api": "LASResNet.stream_host: pinned host image batch -> H2D -> forward (CUDA graph) -> logits "
                           "D2H, H2D of step i+1 overlapping the forward of step i; one event pair around K steps"},
            "stats": {"active_cells_per_block": [int(a) for a in net["act_all"]],
                      "r_patch_per_block": [round(v, 4) for v in r_blocks],
                      "rank_ms_per_step": {"min": round(min(net["rank_ms"]), 4), "max": round(max(net["rank_ms"]), 4),
                                           "mean": round(statistics.fmean(net["rank_ms"]), 4)}},
            "gpu_launches": net["launches_per_step"] * K,
            "clocks": clocks,
        }
        if blk is not None:
            bl = blk
            bms = b_max / K
            dom = max(bl["kern_ms"], key=lambda k: bl["kern_ms"][k])
            broof = roofline_entry(bl["kwork"][dom], bl["kern_ms"][dom], hbm, tfl)
            traffic, tsrc = ncu_traffic(dom, scope="block")
            broof.update({"kernel": dom, "traffic": traffic, "traffic_source": tsrc,
                          "algorithmic": bl["kwork"][dom],
                          "share_of_step": round(bl["kern_ms"][dom] / sum(bl["kern_ms"].values()), 3)})
            t_r = t_roof_ms(bl["bwork"], hbm, tfl)
            block_obj = {
                "workload": WORKLOAD_NAME if (args.hw, args.c_in, args.c_mid) == (28, 512, 128) else
                f"experiment: identity dyn-block {args.hw}x{args.hw}x{args.c_in} c_mid={args.c_mid}",
                "S": args.s, "r_target": args.r, "r_patch": round(bl["stats"]["r_patch"], 4),
                "schedule": "fused" if bl["sched"] == 1 else "separate",
                "ms_per_step": round(bms, 4), "images_per_s": round(args.n * world / (bms * 1e-3), 1),
                "latency_ms": {"p10": round(float(np.percentile(bl["step_ms"], 10)), 4),
                               "p50": round(float(np.percentile(bl["step_ms"], 50)), 4),
                               "p90": round(float(np.percentile(bl["step_ms"], 90)), 4)},
                "kernels_ms": {k: round(v, 4) for k, v in bl["kern_ms"].items()},
                "roofline": broof,
                "kernels_roofline": {k: roofline_entry(bl["kwork"][k], v, hbm, tfl) for k, v in bl["kern_ms"].items()},
                "block_roofline": {"t_roof_ms": round(t_r, 4), "frac": round(t_r / bms, 4),
                                   "definition": "SURVEY 8(d) headline: masker read of x + idx + halo gather + "
                                                 "residual + y + weights; halo-method FLOPs"},
                "dense_ms_per_step": round(b_dense, 4), "speedup_vs_dense": round(b_dense / bms, 3),
                "e2e": {"value": round(args.n * world * K / (b_e2e * 1e-3), 1), "unit": "images/s",
                        "h2d_bytes_per_step": bl["bytes_io"], "d2h_bytes_per_step": bl["bytes_io"]},
                "gpu_launches_per_step": bl["n_launch"],
                "timing": "CUDA events around each CUDA-graph replay, L2 flushed (256 MiB read) and input restored "
                          "before each (untimed); mean of K",
            }
            if world == 1 and not args.no_cpu_baseline:
                block_obj["cpu_baseline"] = cpu_baseline_block(bl["x_cpu"], bl["wts_cpu"], bl["wm_cpu"], bl["blk"].bm,
                                                               args.s, args.cpu_budget, args.n)
            line["block"] = block_obj
        if sweep is not None:
            line["block_sweep"] = sweep
        if coco is not None:
            line["coco_backbone"] = coco
        if regnet is not None:
            line["regnet"] = regnet
        if c1 is not None:
            line["config1"] = c1
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_net(net["x_cpu"], net["weights"], net["net"].oracle_meta(),
                                                    args.cpu_budget)
        if args.detail:
            with open(args.detail, "w") as f:
                json.dump({"line": line, "network_launches": [{k: v for k, v in l.items()} for l in net["launches"]],
                           "step_ms": net["step_ms"]}, f, indent=1, default=str)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch(args):
    """--gpus N > 1 outside torchrun: one process per GPU under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29511"),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_lasnet(args)


if __name__ == "__main__":
    main()
