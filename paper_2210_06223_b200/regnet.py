"""LAS-RegNetY (BASELINE configs[3]): the Y-block with grouped
3x3 and squeeze-and-excitation, dynamic identity blocks and static first
blocks, assembled into RegNetY-800MF.  Marshalling only: every step runs in
liblasnet.so (lasnet_regnet_block, lasnet_regnet_stem, lasnet_head, masker).

Widths are zero-padded to multiples of 64 (synth.pad64): RegNetY-800MF's 32 / 144
/ 784 channels run as 64 / 192 / 832 with zero weights on the extra channels,
which leaves the real channels' values unchanged (tests/test_oracle_regnet.py).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .block import _p, _stream, grid

# torchvision regnet_y_800mf: stem 32; stages (width, depth) = (64, 1), (144, 3), (320, 8),
# (784, 2); group width 16; SE ratio 0.25 of the block input width; stride 2 per stage
REGNET_Y_800MF = dict(stem=32, widths=(64, 144, 320, 784), depths=(1, 3, 8, 2), group_width=16, se_ratio=0.25)


def pad64(c: int) -> int:
    """Channel count rounded up to the tensor-core K-block of 64 (zero channels)."""
    return -(-c // 64) * 64


class RegNetBlock:
    """One Y-block with device-resident weights and preallocated buffers.  Dynamic
    (identity, masker weights given) runs in place; static (first blocks) writes
    self.y."""

    def __init__(self, n, h_in, w_in, c_in, c_out, stride, wts, s=1, dynamic=False, device="cuda",
                 schedule=_lib.SCHED_FUSED):
        self.wts = {k: v.to(device).contiguous() for k, v in wts.items()}
        self.dynamic, self.stride, self.s, self.schedule = dynamic, stride, s, schedule
        self.h, self.w = h_in // stride, w_in // stride
        c_mid = self.wts["wa"].shape[0]
        self.c_out = c_out
        self.desc = _lib.BlockDesc(n, self.h, self.w, c_in, c_mid, c_out, stride, s, _lib.LASNET_BF16)
        W = self.wts
        self.rw = _lib.RegnetWeights(
            W["wa"].data_ptr(), W["ba"].data_ptr(), W["wb"].data_ptr(), W["bb"].data_ptr(), W["se_w1"].data_ptr(),
            W["se_b1"].data_ptr(), W["se_w2"].data_ptr(), W["se_b2"].data_ptr(), W["se_w1"].shape[0],
            W["wc"].data_ptr(), W["bc"].data_ptr(), W["wd"].data_ptr() if "wd" in W else None,
            W["bd"].data_ptr() if "bd" in W else None)
        lib = _lib.load()
        self.ws = torch.zeros(max(lib.lasnet_regnet_workspace_bytes(ctypes.byref(self.desc), int(dynamic)), 1),
                              dtype=torch.uint8, device=device)
        gh, gw = grid(self.h, self.w, s)
        self.ncells = n * gh * gw
        self.bm = 0.0
        if dynamic:
            self.wm = W["wm"].float().contiguous()
            self.mask_buf = torch.empty((n, gh, gw), dtype=torch.uint8, device=device)
            self.logits = torch.empty((n, gh, gw), dtype=torch.float64, device=device)
            self.idx = torch.empty(max(self.ncells, 1), dtype=torch.int32, device=device)
            self.count = torch.zeros(1, dtype=torch.int32, device=device)
            self.mask_desc = _lib.BlockDesc(n, self.h, self.w, c_in, c_in, c_in, 1, s, _lib.LASNET_BF16)
        else:
            self.y = torch.empty((n, self.h, self.w, c_out), dtype=torch.bfloat16, device=device)

    def forward(self, x, y=None):
        lib = _lib.load()
        if self.dynamic:
            y = x if y is None else y
            _lib.check("lasnet_regnet_block", lib.lasnet_regnet_block(
                ctypes.byref(self.desc), ctypes.byref(self.rw), _p(x), _p(y), _p(self.wm), self.bm, self.schedule,
                _p(self.mask_buf), _p(self.idx), _p(self.count), _p(self.ws), self.ws.numel(), _stream()))
            return y
        _lib.check("lasnet_regnet_block", lib.lasnet_regnet_block(
            ctypes.byref(self.desc), ctypes.byref(self.rw), _p(x), _p(self.y), None, 0.0, 0, None, None, None,
            _p(self.ws), self.ws.numel(), _stream()))
        return self.y

    def calibrate_bias(self, x: torch.Tensor, r: float) -> float:
        """Masker bias placing ~r of the cells above threshold on x (as DynBlock)."""
        lib = _lib.load()
        _lib.check("lasnet_mask", lib.lasnet_mask(ctypes.byref(self.mask_desc), _p(x), _p(self.wm), 0.0,
                                                  _p(self.mask_buf), _p(self.logits), _stream()))
        lg = self.logits.flatten().double().sort().values.cpu()
        G = lg.numel()
        k = int(round(r * G))
        if k <= 0:
            b = -(float(lg[-1]) + 1.0)
        elif k >= G:
            b = -(float(lg[0]) - 1.0)
        else:
            b = -0.5 * (float(lg[G - k - 1]) + float(lg[G - k]))
        self.bm = float(torch.tensor(b, dtype=torch.float32))
        return self.bm


class LASRegNet:
    """LAS-RegNetY forward on n images (stem layout [n][H][W + 8][8], as LASResNet):
    RegNet stem (3x3/2) -> 4 stages (static first block with stride 2, dynamic
    identity Y-blocks at S_net) -> global average pool + classifier."""

    def __init__(self, n, weights, hw=224, cfg=None, s_net=(4, 4, 2, 1), device="cuda"):
        cfg = cfg or REGNET_Y_800MF
        H, W = (hw, hw) if isinstance(hw, int) else tuple(hw)
        self.n, self.H, self.W, self.cfg, self.s_net = n, H, W, cfg, tuple(s_net)
        self.depths = tuple(cfg["depths"])
        self.stem_w = weights["stem_w"].to(device).contiguous()
        self.stem_b = weights["stem_b"].to(device).contiguous()
        self.stem_c = cfg["stem"]
        h, w = H // 2, W // 2
        self.stem_y = torch.empty((n, h, w, pad64(cfg["stem"])), dtype=torch.bfloat16, device=device)
        c_in = pad64(cfg["stem"])
        self.stages = []
        for si, (width, depth, s) in enumerate(zip(cfg["widths"], cfg["depths"], s_net)):
            c_out = pad64(width)
            first = RegNetBlock(n, h, w, c_in, c_out, 2, weights[f"s{si}_b0"], device=device)
            h, w = h // 2, w // 2
            dyn = [RegNetBlock(n, h, w, c_out, c_out, 1, weights[f"s{si}_b{b}"], s=s, dynamic=True, device=device)
                   for b in range(1, depth)]
            self.stages.append((first, dyn))
            c_in = c_out
        lib = _lib.load()
        self.fc_w = weights["fc_w"].to(device).contiguous()
        self.fc_b = weights["fc_b"].to(device).contiguous()
        self.head_ws = torch.empty(max(lib.lasnet_head_workspace_bytes(n, c_in), 1), dtype=torch.uint8, device=device)
        self.logits = torch.empty((n, self.fc_w.shape[0]), dtype=torch.float32, device=device)
        self.c_last, self.h_last, self.w_last = c_in, h, w

    def blocks(self):
        for _, dyn in self.stages:
            yield from dyn

    def oracle_meta(self):
        bm = {}
        for si, (_, dyn) in enumerate(self.stages):
            for bi, b in enumerate(dyn):
                bm[f"s{si}_b{bi + 1}"] = float(b.bm)
        return {"depths": self.depths, "s_net": self.s_net, "bm": bm}

    def forward(self, x_pad, calibrate_r=None, dense=False, trace=None):
        """Logits [n, classes].  dense: the comparator (every identity block static,
        out of place -- the same weights without masks)."""
        lib = _lib.load()
        n = self.n
        self.launches = 0

        def mark(kind, obj=None, **kw):
            if trace is not None:
                trace.append(dict(kind=kind, obj=obj, ev1=int(lib.lasnet_kernel_event_count()), **kw))
            self.launches += int(lib.lasnet_last_launch_count())

        _lib.check("lasnet_regnet_stem", lib.lasnet_regnet_stem(n, self.H // 2, self.W // 2, self.stem_c, _p(x_pad),
                                                                _p(self.stem_w), _p(self.stem_b), _p(self.stem_y),
                                                                _stream()))
        mark("stem")
        x = self.stem_y
        for si, (first, dyn) in enumerate(self.stages):
            y = first.forward(x)
            mark("proj", first, stage=si)
            for bi, blk in enumerate(dyn):
                if dense:
                    y = self._dense(si, bi, blk).forward(y)
                else:
                    if calibrate_r is not None:
                        blk.calibrate_bias(y, calibrate_r)
                    blk.forward(y)
                mark("dense" if dense else "dyn", blk, stage=si, block=bi + 1)
            x = y
        _lib.check("lasnet_head", lib.lasnet_head(n, self.h_last * self.w_last, self.c_last, self.fc_w.shape[0],
                                                  _p(x), _p(self.fc_w), _p(self.fc_b), _p(self.logits),
                                                  _p(self.head_ws), self.head_ws.numel(), _stream()))
        mark("head")
        if trace is not None:
            for i, t in enumerate(trace):
                t["ev0"] = trace[i - 1]["ev1"] if i else 0
        return self.logits

    def _dense(self, si, bi, blk):
        if not hasattr(self, "_dense_blocks"):
            self._dense_blocks = {}
        key = (si, bi)
        if key not in self._dense_blocks:
            d = blk.desc
            wts = {k: v for k, v in blk.wts.items() if k != "wm"}
            self._dense_blocks[key] = RegNetBlock(d.n, d.h, d.w, d.c_in, d.c_out, 1, wts, device=blk.wts["wa"].device)
        return self._dense_blocks[key]

    def capture(self, x_pad, dense=False):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.forward(x_pad, dense=dense)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward(x_pad, dense=dense)
        return g
