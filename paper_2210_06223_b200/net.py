"""LAS-ResNet forward built from the library's layers.

    stem (7x7/2, tcgen05) -> 3x3/2 max pool -> 4 stages -> global average pool + classifier

Each stage is one static projection block (lasnet_proj_block: the stride-2 /
channel-changing first block, whose shortcut LASNet keeps dense) followed
by the stage's identity blocks as dynamic blocks (lasnet_block_forward: masker
-> compaction -> gather + conv1 -> conv2 -> conv3 + scatter-add, in place) at
the stage's granularity S (S_net 4-4-2-1).  ResNet-101: depths
3-4-23-3, bottleneck widths 64-128-256-512 (x4 outputs).

Every buffer is allocated once at construction, so ``forward`` is only kernel
launches (no host synchronisation) and can be captured in one CUDA graph.  This
module only marshals: all arithmetic runs in liblasnet.so.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .block import BlockShape, DynBlock, ProjDynBlock, _p, _stream, choose_schedule

R101_DEPTHS = (3, 4, 23, 3)
R50_DEPTHS = (3, 4, 6, 3)
WIDTHS = (64, 128, 256, 512)
S_NET = (4, 4, 2, 1)


class ProjBlock:
    """Static projection block with preallocated output and workspace."""

    def __init__(self, n, h_in, w_in, c_in, c_mid, c_out, stride, wts, device="cuda"):
        self.wts = {k: v.to(device).contiguous() for k, v in wts.items()}
        self.h, self.w = h_in // stride, w_in // stride
        self.desc = _lib.BlockDesc(n, self.h, self.w, c_in, c_mid, c_out, stride, 1, _lib.LASNET_BF16)
        self.wt = _lib.BlockWeights(*(self.wts[k].data_ptr() for k in ("w1", "b1", "w2", "b2", "w3", "b3", "wd", "bd")))
        lib = _lib.load()
        self.ws = torch.empty(max(lib.lasnet_proj_workspace_bytes(ctypes.byref(self.desc)), 1), dtype=torch.uint8,
                              device=device)
        self.y = torch.empty((n, self.h, self.w, c_out), dtype=torch.bfloat16, device=device)

    def forward(self, x):
        _lib.check("lasnet_proj_block", _lib.load().lasnet_proj_block(
            ctypes.byref(self.desc), ctypes.byref(self.wt), _p(x), _p(self.y), _p(self.ws), self.ws.numel(),
            _stream()))
        return self.y


class LASResNet:
    """LAS-ResNet forward on a batch of n images of H x W (hw: an int for square
    ImageNet input, or (H, W), e.g. the COCO backbone's 800 x 1344; 3 channels
    zero-padded to 8, given as the stem's padded layout [n][H][W + 8][8]).
    backbone=True stops after the last stage (detection-shaped feature maps,
    BASELINE configs[4]): forward returns the four stage outputs."""

    def __init__(self, n: int, weights: dict, hw=224, depths=R101_DEPTHS, s_net=S_NET, r: float = 0.5,
                 device="cuda", dynamic_proj: bool = True, backbone: bool = False):
        H, W = (hw, hw) if isinstance(hw, int) else tuple(hw)
        if H % 32 or W % 32:
            raise ValueError("input height and width must be multiples of 32")
        self.n, self.hw, self.H, self.W, self.device = n, hw, H, W, device
        self.backbone = backbone
        self.depths, self.s_net = tuple(depths), tuple(s_net)
        lib = _lib.load()
        self.stem_w = weights["stem_w"].to(device).contiguous()
        self.stem_b = weights["stem_b"].to(device).contiguous()
        self.stem_ws = torch.empty(lib.lasnet_stem_workspace_bytes(), dtype=torch.uint8, device=device)
        h, w = H // 2, W // 2
        self.stem_y = torch.empty((n, h, w, 64), dtype=torch.bfloat16, device=device)
        h, w = h // 2, w // 2
        self.pool_y = torch.empty((n, h, w, 64), dtype=torch.bfloat16, device=device)
        self.stages = []
        self.static_proj = []
        c_in = 64
        for si, (depth, width, s) in enumerate(zip(depths, WIDTHS, s_net)):
            stride = 1 if si == 0 else 2
            c_out = 4 * width
            pw = weights[f"s{si}_proj"]
            static = ProjBlock(n, h, w, c_in, width, c_out, stride, pw, device)  # the dense comparator's
            proj = (ProjDynBlock(n, h, w, c_in, width, c_out, stride, s, pw, pw["wm"], 0.0, device)
                    if dynamic_proj else static)
            self.static_proj.append(static)
            h, w = h // stride, w // stride
            dyn = []
            for b in range(1, depth):
                wb = weights[f"s{si}_b{b}"]
                sched = choose_schedule(n, h, w, c_out, width, c_out, s, r)
                dyn.append(DynBlock(BlockShape(n, h, w, c_out, width, s), {k: wb[k] for k in
                                                                           ("w1", "b1", "w2", "b2", "w3", "b3")},
                                    wb["wm"], 0.0, device=device, schedule=sched))
            self.stages.append((proj, dyn))
            c_in = c_out
        self.fc_w = weights["fc_w"].to(device).contiguous()
        self.fc_b = weights["fc_b"].to(device).contiguous()
        self.head_ws = torch.empty(max(lib.lasnet_head_workspace_bytes(n, c_in), 1), dtype=torch.uint8,
                                   device=device)
        self.logits = torch.empty((n, self.fc_w.shape[0]), dtype=torch.float32, device=device)
        self.c_last, self.h_last, self.w_last = c_in, h, w
        self.features = [None] * len(self.stages)

    def oracle_meta(self) -> dict:
        """Depths, S_net and every dynamic block's masker bias, keyed like the weight
        dict ("s{stage}_b{block}") -- what an oracle forward needs to take the same
        decisions (test / bench bookkeeping; no arithmetic)."""
        bm = {}
        for si, (proj, dyn) in enumerate(self.stages):
            if getattr(proj, "dynamic", False):
                bm[f"s{si}_proj"] = float(proj.bm)
            for bi, blk in enumerate(dyn):
                bm[f"s{si}_b{bi + 1}"] = float(blk.bm)
        return {"depths": self.depths, "s_net": self.s_net, "bm": bm,
                "dyn_proj": all(getattr(p, "dynamic", False) for p, _ in self.stages)}

    def blocks(self):
        """Every dynamic block in forward order (the dynamic first blocks included)."""
        for proj, dyn in self.stages:
            if getattr(proj, "dynamic", False):
                yield proj
            yield from dyn

    def forward(self, x_pad: torch.Tensor, calibrate_r: float | None = None, dense: bool = False,
                trace: list | None = None):
        """Logits [n, classes] (fp32).  calibrate_r: first set every dynamic block's
        masker bias so that ~r of its cells are active on the activations it sees
        (host synchronisation; not for the timed path).  dense: run the identity
        blocks on every pixel (lasnet_dense_block) -- the comparator network.
        trace: if a list, one dict per library call is appended (layer kind, the
        block object, and the range [ev0, ev1) of kernel event pairs the call
        recorded when lasnet_set_kernel_events is armed) -- bench bookkeeping."""
        lib = _lib.load()
        n, h, w = self.n, self.H // 2, self.W // 2
        self.launches = 0

        def mark(kind, obj=None, **kw):
            if trace is not None:
                trace.append(dict(kind=kind, obj=obj, ev1=int(lib.lasnet_kernel_event_count()), **kw))
            self.launches += int(lib.lasnet_last_launch_count())

        _lib.check("lasnet_stem", lib.lasnet_stem(n, h, w, _p(x_pad), _p(self.stem_w), _p(self.stem_b),
                                                  _p(self.stem_y), _p(self.stem_ws), self.stem_ws.numel(), _stream()))
        mark("stem", None, n=n, h=h, w=w)
        _lib.check("lasnet_maxpool", lib.lasnet_maxpool(n, h // 2, w // 2, 64, _p(self.stem_y), _p(self.pool_y),
                                                        _stream()))
        mark("maxpool", None, n=n, h=h // 2, w=w // 2, c=64)
        x = self.pool_y
        for si, (proj, dyn) in enumerate(self.stages):
            if dense:
                proj = self.static_proj[si]
            elif calibrate_r is not None and getattr(proj, "dynamic", False):
                proj.calibrate_bias(x, calibrate_r)
            y = proj.forward(x)
            mark("proj", proj, stage=si)
            other = self._scratch(si, y) if dense else None
            for bi, blk in enumerate(dyn):
                if calibrate_r is not None:
                    blk.calibrate_bias(y, calibrate_r)
                if dense:  # out of place, ping-pong between the stage's two buffers
                    blk.dense(y, other)
                    y, other = other, y
                else:
                    blk.forward(y)  # in place: inactive pixels are never touched
                mark("dense" if dense else "dyn", blk, stage=si, block=bi + 1)
            self.features[si] = y
            x = y
        if not self.backbone:
            _lib.check("lasnet_head", lib.lasnet_head(n, self.h_last * self.w_last, self.c_last, self.fc_w.shape[0],
                                                      _p(x), _p(self.fc_w), _p(self.fc_b), _p(self.logits),
                                                      _p(self.head_ws), self.head_ws.numel(), _stream()))
            mark("head", None, n=n, hw=self.h_last * self.w_last, c=self.c_last, classes=self.fc_w.shape[0])
        if trace is not None:  # ev0 of each call = ev1 of the previous one
            for i, t in enumerate(trace):
                t["ev0"] = trace[i - 1]["ev1"] if i else 0
        return list(self.features) if self.backbone else self.logits

    def stream_host(self, x_hosts, logits_hosts, x_devs, graphs, steps: int):
        """End-to-end serving loop with HOST buffers (e2e of bench.py): step i copies
        the pinned image batch x_hosts[i % len] into x_devs[i % 2] on an H2D stream,
        replays graphs[i % 2] (the forward captured on that input buffer) on the
        current stream and copies the logits into logits_hosts[i % len] (pinned) on a
        D2H stream; the H2D of step i+1 overlaps the forward of step i.  Enqueues
        everything; the current stream then waits for the last D2H."""
        comp = torch.cuda.current_stream()
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = (torch.cuda.Stream(), torch.cuda.Stream())
        h2d, d2h = self._copy_streams
        h2d.wait_stream(comp)
        d2h.wait_stream(comp)
        nb = len(x_devs)
        freed = [None] * nb  # the forward that read x_devs[b] has finished: it may be overwritten
        out_done = None
        for i in range(steps):
            b = i % nb
            with torch.cuda.stream(h2d):
                if freed[b] is not None:
                    h2d.wait_event(freed[b])
                x_devs[b].copy_(x_hosts[i % len(x_hosts)], non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(h2d)
            comp.wait_event(loaded)
            if out_done is not None:
                comp.wait_event(out_done)  # the previous step's logits have been read out
            graphs[b].replay()
            done = torch.cuda.Event()
            done.record(comp)
            freed[b] = done
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                logits_hosts[i % len(logits_hosts)].copy_(self.logits, non_blocking=True)
                out_done = torch.cuda.Event()
                out_done.record(d2h)
        comp.wait_stream(h2d)
        comp.wait_stream(d2h)
        return logits_hosts

    def _scratch(self, si, like):
        if not hasattr(self, "_scr"):
            self._scr = {}
        if si not in self._scr:
            self._scr[si] = torch.empty_like(like)
        return self._scr[si]

    def capture(self, x_pad: torch.Tensor, dense: bool = False) -> torch.cuda.CUDAGraph:
        """The whole forward as one CUDA graph on these buffers."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.forward(x_pad, dense=dense)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward(x_pad, dense=dense)
        return g
