"""Python API of the LASNet dynamic residual block (thin marshalling over the C ABI).

Every step of the block runs in liblasnet.so kernels; this module only creates
descriptor structs, allocates caller-owned buffers with torch and passes raw
device pointers plus the current CUDA stream.  Functions mirror the C-ABI
names: ``mask``, ``compact``, ``dyn_block``, ``dense_block``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import SCHED_SEPARATE

_DT = {torch.bfloat16: _lib.LASNET_BF16, torch.float32: _lib.LASNET_F32}


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def grid(h: int, w: int, s: int):
    return -(-h // s), -(-w // s)


def make_desc(n, h, w, c_in, c_mid, c_out, s, dtype) -> _lib.BlockDesc:
    return _lib.BlockDesc(n, h, w, c_in, c_mid, c_out, 1, s, _DT[dtype])


def make_weights(wts: dict) -> _lib.BlockWeights:
    return _lib.BlockWeights(*(wts[k].data_ptr() for k in ("w1", "b1", "w2", "b2", "w3", "b3")), None, None)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("lasnet: tensors must be contiguous CUDA tensors")


# ------------------------------------------------------------- functional --

def mask(x: torch.Tensor, wm: torch.Tensor, bm: float, s: int, logits: bool = False,
         out: torch.Tensor | None = None, logits_out: torch.Tensor | None = None):
    """Step 1: uint8 [n, gh, gw] mask and optional fp64 logits."""
    _require_cuda(x, wm)
    n, h, w, c = x.shape
    gh, gw = grid(h, w, s)
    m = out if out is not None else torch.empty((n, gh, gw), dtype=torch.uint8, device=x.device)
    lg = logits_out if logits_out is not None else (
        torch.empty((n, gh, gw), dtype=torch.float64, device=x.device) if logits else None)
    d = make_desc(n, h, w, c, c, c, s, x.dtype)
    lib = _lib.load()
    _lib.check("lasnet_mask", lib.lasnet_mask(ctypes.byref(d), _p(x), _p(wm), float(bm), _p(m), _p(lg), _stream()))
    return (m, lg) if logits else m


def compact(m: torch.Tensor, idx: torch.Tensor | None = None, count: torch.Tensor | None = None,
            ws: torch.Tensor | None = None):
    """Step 2: ascending active cell ids + device count."""
    _require_cuda(m)
    lib = _lib.load()
    ncells = m.numel()
    idx = idx if idx is not None else torch.empty(max(ncells, 1), dtype=torch.int32, device=m.device)
    count = count if count is not None else torch.empty(1, dtype=torch.int32, device=m.device)
    wsb = lib.lasnet_compact_workspace_bytes(ncells)
    ws = ws if ws is not None else torch.empty(wsb, dtype=torch.uint8, device=m.device)
    _lib.check("lasnet_compact", lib.lasnet_compact(_p(m), ncells, _p(idx), _p(count), _p(ws), ws.numel(), _stream()))
    return idx, count


def dyn_block(x: torch.Tensor, wts: dict, idx: torch.Tensor, count: torch.Tensor, s: int,
              y: torch.Tensor | None = None, ws: torch.Tensor | None = None, cap: int | None = None):
    """Steps 3-5.  y=None runs in place on x."""
    _require_cuda(x, idx, count)
    lib = _lib.load()
    n, h, w, c_in = x.shape
    c_mid, c_out = wts["w1"].shape[0], wts["w3"].shape[0]
    gh, gw = grid(h, w, s)
    cap = cap if cap is not None else n * gh * gw
    d = make_desc(n, h, w, c_in, c_mid, c_out, s, x.dtype)
    wsb = lib.lasnet_dyn_workspace_bytes(ctypes.byref(d), cap)
    ws = ws if ws is not None else torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    y = x if y is None else y
    wt = make_weights(wts)
    _lib.check("lasnet_dyn_block", lib.lasnet_dyn_block(ctypes.byref(d), ctypes.byref(wt), _p(x), _p(y), _p(idx),
                                                        _p(count), cap, _p(ws), ws.numel(), _stream()))
    return y


def dense_block(x: torch.Tensor, wts: dict, y: torch.Tensor | None = None, ws: torch.Tensor | None = None):
    """Static comparator: the same kernels on every pixel."""
    _require_cuda(x)
    lib = _lib.load()
    n, h, w, c_in = x.shape
    c_mid, c_out = wts["w1"].shape[0], wts["w3"].shape[0]
    d = make_desc(n, h, w, c_in, c_mid, c_out, 1, x.dtype)
    wsb = lib.lasnet_dense_workspace_bytes(ctypes.byref(d))
    ws = ws if ws is not None else torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    y = torch.empty_like(x) if y is None else y
    wt = make_weights(wts)
    _lib.check("lasnet_dense_block", lib.lasnet_dense_block(ctypes.byref(d), ctypes.byref(wt), _p(x), _p(y), _p(ws),
                                                            ws.numel(), _stream()))
    return y


def proj_block(x: torch.Tensor, wts: dict, stride: int, ws: torch.Tensor | None = None):
    """Static projection (first) block of a stage (lasnet_proj_block; NEXT-f1):
    x [n, h*stride, w*stride, c_in] -> y [n, h, w, c_out] with the 1x1 stride-s
    shortcut wts["wd"] [c_out][c_in], wts["bd"] [c_out]."""
    _require_cuda(x)
    lib = _lib.load()
    n, hi, wi, c_in = x.shape
    c_mid, c_out = wts["w1"].shape[0], wts["w3"].shape[0]
    if hi % stride or wi % stride:
        raise ValueError("input size must be a multiple of the stride")
    h, w = hi // stride, wi // stride
    d = _lib.BlockDesc(n, h, w, c_in, c_mid, c_out, stride, 1, _DT[x.dtype])
    wsb = lib.lasnet_proj_workspace_bytes(ctypes.byref(d))
    ws = ws if ws is not None else torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    y = torch.empty((n, h, w, c_out), dtype=x.dtype, device=x.device)
    wt = _lib.BlockWeights(*(wts[k].data_ptr() for k in ("w1", "b1", "w2", "b2", "w3", "b3", "wd", "bd")))
    _lib.check("lasnet_proj_block", lib.lasnet_proj_block(ctypes.byref(d), ctypes.byref(wt), _p(x), _p(y), _p(ws),
                                                          ws.numel(), _stream()))
    return y


def stem(x_pad: torch.Tensor, w: torch.Tensor, b: torch.Tensor, ws: torch.Tensor | None = None):
    """7x7 stride-2 stem (lasnet_stem): x_pad [n, 2h, 2w + 8, 8] (3 channels zero-padded
    to 8, 4 zero pixels left and right) -> y [n, h, w, 64]."""
    _require_cuda(x_pad, w, b)
    lib = _lib.load()
    n, hi, wp, c = x_pad.shape
    h, w_out = hi // 2, (wp - 8) // 2
    ws = ws if ws is not None else torch.empty(lib.lasnet_stem_workspace_bytes(), dtype=torch.uint8,
                                               device=x_pad.device)
    y = torch.empty((n, h, w_out, 64), dtype=x_pad.dtype, device=x_pad.device)
    _lib.check("lasnet_stem", lib.lasnet_stem(n, h, w_out, _p(x_pad), _p(w), _p(b), _p(y), _p(ws), ws.numel(),
                                              _stream()))
    return y


def maxpool(x: torch.Tensor):
    """3x3 stride-2 max pool, padding 1 (lasnet_maxpool): [n, 2h, 2w, c] -> [n, h, w, c]."""
    _require_cuda(x)
    n, hi, wi, c = x.shape
    y = torch.empty((n, hi // 2, wi // 2, c), dtype=x.dtype, device=x.device)
    _lib.check("lasnet_maxpool", _lib.load().lasnet_maxpool(n, hi // 2, wi // 2, c, _p(x), _p(y), _stream()))
    return y


def head(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor, ws: torch.Tensor | None = None):
    """Global average pool + classifier (lasnet_head): x [n, h, w, c] -> fp32 logits [n, classes]."""
    _require_cuda(x, w, b)
    lib = _lib.load()
    n, h, wd, c = x.shape
    classes = w.shape[0]
    ws = ws if ws is not None else torch.empty(max(lib.lasnet_head_workspace_bytes(n, c), 1), dtype=torch.uint8,
                                               device=x.device)
    logits = torch.empty((n, classes), dtype=torch.float32, device=x.device)
    _lib.check("lasnet_head", lib.lasnet_head(n, h * wd, c, classes, _p(x), _p(w), _p(b), _p(logits), _p(ws),
                                              ws.numel(), _stream()))
    return logits


def block_forward(x: torch.Tensor, wts: dict, wm: torch.Tensor, bm: float, s: int, schedule: int,
                  y: torch.Tensor | None = None, ws: torch.Tensor | None = None, mask_out: bool = True):
    """Steps 1-5 in one C-ABI call (lasnet_block_forward) under `schedule`
    (SCHED_SEPARATE: the north-star branch; SCHED_FUSED: the paper's Table-1
    schedule, masker fused into a static conv1).  Returns (y, mask, idx, count).
    y=None runs in place on x."""
    _require_cuda(x, wm)
    lib = _lib.load()
    n, h, w, c_in = x.shape
    c_mid, c_out = wts["w1"].shape[0], wts["w3"].shape[0]
    gh, gw = grid(h, w, s)
    d = make_desc(n, h, w, c_in, c_mid, c_out, s, x.dtype)
    wsb = lib.lasnet_block_forward_workspace_bytes(ctypes.byref(d), schedule)
    ws = ws if ws is not None else torch.zeros(max(wsb, 1), dtype=torch.uint8, device=x.device)
    y = x if y is None else y
    m = torch.empty((n, gh, gw), dtype=torch.uint8, device=x.device) if mask_out else None
    idx = torch.empty(max(n * gh * gw, 1), dtype=torch.int32, device=x.device)
    count = torch.empty(1, dtype=torch.int32, device=x.device)
    wt = make_weights(wts)
    _lib.check("lasnet_block_forward", lib.lasnet_block_forward(
        ctypes.byref(d), ctypes.byref(wt), _p(x), _p(y), _p(wm), float(bm), int(schedule), _p(m), _p(idx),
        _p(count), _p(ws), ws.numel(), _stream()))
    return y, m, idx, count


def proj_block_forward(x: torch.Tensor, wts: dict, wm: torch.Tensor, bm: float, s: int, stride: int,
                       ws: torch.Tensor | None = None):
    """The dynamic projection (first) block of a stage, steps 1-5 in one C-ABI call
    (lasnet_block_forward with the shortcut weights wts["wd"], wts["bd"]; NEXT-f1,
    DESIGN.md reading R22): x [n, h*stride, w*stride, c_in] -> y [n, h, w, c_out]
    with y = ReLU(R + M F(x)), R = Wd x_s + bd computed densely, the mask on the
    output grid from the masker pooling each cell's stride*S input window.
    Returns (y, mask, idx, count)."""
    _require_cuda(x, wm)
    lib = _lib.load()
    n, hi, wi, c_in = x.shape
    c_mid, c_out = wts["w1"].shape[0], wts["w3"].shape[0]
    if hi % stride or wi % stride:
        raise ValueError("input size must be a multiple of the stride")
    h, w = hi // stride, wi // stride
    gh, gw = grid(h, w, s)
    d = _lib.BlockDesc(n, h, w, c_in, c_mid, c_out, stride, s, _DT[x.dtype])
    wsb = lib.lasnet_block_forward_workspace_bytes(ctypes.byref(d), SCHED_SEPARATE)
    ws = ws if ws is not None else torch.zeros(max(wsb, 1), dtype=torch.uint8, device=x.device)
    y = torch.empty((n, h, w, c_out), dtype=x.dtype, device=x.device)
    m = torch.empty((n, gh, gw), dtype=torch.uint8, device=x.device)
    idx = torch.empty(max(n * gh * gw, 1), dtype=torch.int32, device=x.device)
    count = torch.empty(1, dtype=torch.int32, device=x.device)
    wt = _lib.BlockWeights(*(wts[k].data_ptr() for k in ("w1", "b1", "w2", "b2", "w3", "b3", "wd", "bd")))
    _lib.check("lasnet_block_forward", lib.lasnet_block_forward(
        ctypes.byref(d), ctypes.byref(wt), _p(x), _p(y), _p(wm), float(bm), SCHED_SEPARATE, _p(m), _p(idx),
        _p(count), _p(ws), ws.numel(), _stream()))
    return y, m, idx, count


def predict_latency(n, h, w, c_in, c_mid, c_out, s, r, schedule, stride: int = 1, hw=None):
    """lasnet_predict_latency (the B200 latency predictor G(H, P, S, r)):
    (total_us, [(kernel type, us), ...]) of one block call; schedule SCHED_SEPARATE,
    SCHED_FUSED or SCHED_DENSE (the static block); h, w the output dims.  hw: an
    _lib.HW (None = the built-in B200 calibration)."""
    lib = _lib.load()
    d = _lib.BlockDesc(n, h, w, c_in, c_mid, c_out, stride, s, _lib.LASNET_BF16)
    kinds = (ctypes.c_int32 * 8)()
    us = (ctypes.c_double * 8)()
    nk = ctypes.c_int32(0)
    t = lib.lasnet_predict_latency(ctypes.byref(d), int(schedule), float(r), ctypes.byref(hw) if hw else None,
                                   kinds, us, 8, ctypes.byref(nk))
    if t < 0:
        raise ValueError("lasnet_predict_latency: invalid arguments or unsupported schedule")
    return t, [(lib.lasnet_kernel_type_name(kinds[i]).decode(), us[i]) for i in range(nk.value)]


def hw_b200():
    """The predictor's built-in B200 hardware model (an _lib.HW to modify)."""
    h = _lib.HW()
    _lib.load().lasnet_hw_b200(ctypes.byref(h))
    return h


def choose_schedule(n, h, w, c_in, c_mid, c_out, s, r, dtype=torch.bfloat16) -> int:
    d = make_desc(n, h, w, c_in, c_mid, c_out, s, dtype)
    return int(_lib.load().lasnet_choose_schedule(ctypes.byref(d), float(r)))


def last_launch_count() -> int:
    return int(_lib.load().lasnet_last_launch_count())


# ------------------------------------------------------------------ block --

@dataclass
class BlockShape:
    n: int
    h: int
    w: int
    c_in: int
    c_mid: int
    s: int
    dtype: torch.dtype = torch.bfloat16

    @property
    def gh(self):
        return -(-self.h // self.s)

    @property
    def gw(self):
        return -(-self.w // self.s)

    @property
    def ncells(self):
        return self.n * self.gh * self.gw


class DynBlock:
    """One LASNet bottleneck block with device-resident weights and caller-owned
    buffers preallocated once (mask, idx, count, workspaces), so a forward is
    exactly the kernel launches: mask -> compact -> conv1 -> conv2 -> conv3."""

    def __init__(self, shape: BlockShape, wts: dict, wm: torch.Tensor, bm: float, device="cuda",
                 schedule: int | None = None):
        self.shape = shape
        self.wts = {k: v.to(device).contiguous() for k, v in wts.items()}
        self.wm = wm.to(device).float().contiguous()
        self.bm = float(bm)
        sh = shape
        self.c_out = self.wts["w3"].shape[0]
        lib = _lib.load()
        self.desc = make_desc(sh.n, sh.h, sh.w, sh.c_in, sh.c_mid, self.c_out, sh.s, sh.dtype)
        self.wt = make_weights(self.wts)
        self.mask_buf = torch.empty((sh.n, sh.gh, sh.gw), dtype=torch.uint8, device=device)
        self.logits = torch.empty((sh.n, sh.gh, sh.gw), dtype=torch.float64, device=device)
        self.idx = torch.empty(max(sh.ncells, 1), dtype=torch.int32, device=device)
        self.count = torch.zeros(1, dtype=torch.int32, device=device)
        self.cws = torch.empty(max(lib.lasnet_compact_workspace_bytes(sh.ncells), 1), dtype=torch.uint8, device=device)
        # fused masker+compaction workspace: zero before first use, left zero by every call
        self.mcws = torch.zeros(max(lib.lasnet_mask_compact_workspace_bytes(ctypes.byref(self.desc)), 16),
                                dtype=torch.uint8, device=device)
        self.cap = sh.ncells
        self.dws = torch.empty(max(lib.lasnet_dyn_workspace_bytes(ctypes.byref(self.desc), self.cap), 1),
                               dtype=torch.uint8, device=device)
        # schedule: None = the north-star step-by-step calls (mask_compact + dyn_block);
        # SCHED_SEPARATE / SCHED_FUSED = one lasnet_block_forward call
        self.schedule = schedule
        self.fws = None
        if schedule is not None:
            self.fws = torch.zeros(max(lib.lasnet_block_forward_workspace_bytes(ctypes.byref(self.desc), schedule), 1),
                                   dtype=torch.uint8, device=device)
        dd = make_desc(sh.n, sh.h, sh.w, sh.c_in, sh.c_mid, self.c_out, 1, sh.dtype)
        self.dense_desc = dd
        self._dense_ws = None
        self.launches = 0

    @property
    def ncells(self):
        return self.shape.ncells

    def mask(self, x: torch.Tensor, want_logits: bool = False):
        lib = _lib.load()
        _lib.check("lasnet_mask", lib.lasnet_mask(ctypes.byref(self.desc), _p(x), _p(self.wm), self.bm,
                                                  _p(self.mask_buf), _p(self.logits) if want_logits else None,
                                                  _stream()))
        self.launches += lib.lasnet_last_launch_count()
        return self.mask_buf

    def compact(self):
        lib = _lib.load()
        _lib.check("lasnet_compact", lib.lasnet_compact(_p(self.mask_buf), self.shape.ncells, _p(self.idx),
                                                        _p(self.count), _p(self.cws), self.cws.numel(), _stream()))
        self.launches += lib.lasnet_last_launch_count()
        return self.idx, self.count

    def mask_compact(self, x: torch.Tensor, want_logits: bool = False):
        """Steps 1+2 in one launch (lasnet_mask_compact)."""
        lib = _lib.load()
        _lib.check("lasnet_mask_compact", lib.lasnet_mask_compact(
            ctypes.byref(self.desc), _p(x), _p(self.wm), self.bm, _p(self.mask_buf),
            _p(self.logits) if want_logits else None, _p(self.idx), _p(self.count), _p(self.mcws),
            self.mcws.numel(), _stream()))
        self.launches += lib.lasnet_last_launch_count()
        return self.idx, self.count

    def convs(self, x: torch.Tensor, y: torch.Tensor | None = None):
        lib = _lib.load()
        y = x if y is None else y
        _lib.check("lasnet_dyn_block", lib.lasnet_dyn_block(ctypes.byref(self.desc), ctypes.byref(self.wt), _p(x),
                                                            _p(y), _p(self.idx), _p(self.count), self.cap,
                                                            _p(self.dws), self.dws.numel(), _stream()))
        self.launches += lib.lasnet_last_launch_count()
        return y

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None):
        """Five steps, in place on x when y is None.  No host synchronisation.
        schedule None: steps 1+2 as one fused launch, then lasnet_dyn_block;
        otherwise one lasnet_block_forward call under self.schedule."""
        if self.schedule is None:
            self.mask_compact(x)
            return self.convs(x, y)
        lib = _lib.load()
        y = x if y is None else y
        _lib.check("lasnet_block_forward", lib.lasnet_block_forward(
            ctypes.byref(self.desc), ctypes.byref(self.wt), _p(x), _p(y), _p(self.wm), self.bm, self.schedule,
            _p(self.mask_buf), _p(self.idx), _p(self.count), _p(self.fws), self.fws.numel(), _stream()))
        self.launches += lib.lasnet_last_launch_count()
        return y

    __call__ = forward

    def capture(self, x: torch.Tensor, y: torch.Tensor | None = None, warmup: int = 2) -> torch.cuda.CUDAGraph:
        """Capture one forward on these exact buffers into a CUDA graph (the TMA
        descriptors are kernel parameters, so the graph is bound to x / y and the
        block's workspaces; re-capture if they change).  Replaying the graph runs
        the same kernels with one launch call instead of one per kernel."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):  # first calls set kernel attributes outside the capture
                self.forward(x, y)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward(x, y)
        return g

    def dense(self, x: torch.Tensor, y: torch.Tensor):
        lib = _lib.load()
        if self._dense_ws is None:
            self._dense_ws = torch.empty(max(lib.lasnet_dense_workspace_bytes(ctypes.byref(self.dense_desc)), 1),
                                         dtype=torch.uint8, device=x.device)
        _lib.check("lasnet_dense_block", lib.lasnet_dense_block(ctypes.byref(self.dense_desc), ctypes.byref(self.wt),
                                                                _p(x), _p(y), _p(self._dense_ws),
                                                                self._dense_ws.numel(), _stream()))
        self.launches += lib.lasnet_last_launch_count()
        return y

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor):
        """End-to-end call with HOST buffers: H2D copy of x (pinned) into x_dev,
        the five steps in place, D2H copy of the result into y_host (pinned)."""
        x_dev.copy_(x_host, non_blocking=True)
        self.forward(x_dev)
        y_host.copy_(x_dev, non_blocking=True)
        return y_host

    def stream_host(self, x_hosts, y_hosts, x_devs, steps: int, before_step=None):
        """Pipelined end-to-end batches with HOST buffers (a serving loop): step i
        copies x_hosts[i % len] (pinned) into x_devs[i % len(x_devs)] on an H2D
        stream, runs the five steps in place on the current stream, and copies the
        result into y_hosts[i % len] (pinned) on a D2H stream, so the two copy
        directions of neighbouring steps overlap each other and the compute.
        Enqueues everything and returns; the current stream then waits for the
        last D2H.  before_step(i), if given, is enqueued on the compute stream
        before step i (e.g. an L2 flush)."""
        comp = torch.cuda.current_stream()
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = (torch.cuda.Stream(), torch.cuda.Stream())
        h2d, d2h = self._copy_streams
        nb = len(x_devs)
        h2d.wait_stream(comp)
        d2h.wait_stream(comp)
        freed = [None] * nb  # D2H done with x_devs[b]: it may be overwritten
        for i in range(steps):
            b = i % nb
            xd = x_devs[b]
            with torch.cuda.stream(h2d):
                if freed[b] is not None:
                    h2d.wait_event(freed[b])
                xd.copy_(x_hosts[i % len(x_hosts)], non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(h2d)
            comp.wait_event(loaded)
            if before_step is not None:
                before_step(i)
            self.forward(xd)
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                y_hosts[i % len(y_hosts)].copy_(xd, non_blocking=True)
                freed[b] = torch.cuda.Event()
                freed[b].record(d2h)
        comp.wait_stream(h2d)
        comp.wait_stream(d2h)
        return y_hosts

    def calibrate_bias(self, x: torch.Tensor, r: float) -> float:
        """Pick the masker bias so that ~r of the cells are active on x, from the
        product masker's own logits (b = 0): bm = -(the (1-r) quantile), placed
        midway between two neighbouring logits so no cell sits on the threshold."""
        saved = self.bm
        self.bm = 0.0
        self.mask(x, want_logits=True)
        lg = self.logits.flatten().double().sort().values.cpu()
        self.bm = saved
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


class ProjDynBlock:
    """The dynamic projection (first) block of a stage (NEXT-f1, reading R22) with
    device-resident weights and preallocated buffers: x [n, h*stride, w*stride,
    c_in] -> self.y [n, h, w, c_out].  One lasnet_block_forward call per forward:
    masker (stride*S input window per output cell) + compaction, the dense 1x1
    stride-s shortcut, gather + conv1 over the active windows, the stride-s 3x3,
    conv3 + scatter-add onto the shortcut."""

    dynamic = True

    def __init__(self, n, h_in, w_in, c_in, c_mid, c_out, stride, s, wts, wm, bm=0.0, device="cuda"):
        self.wts = {k: v.to(device).contiguous() for k, v in wts.items() if k != "wm"}
        self.wm = wm.to(device).float().contiguous()
        self.bm = float(bm)
        self.stride, self.s = stride, s
        self.h, self.w = h_in // stride, w_in // stride
        self.c_out = c_out
        self.desc = _lib.BlockDesc(n, self.h, self.w, c_in, c_mid, c_out, stride, s, _lib.LASNET_BF16)
        # the masker's view: the input at granularity stride * S (same cell grid)
        self.mask_desc = _lib.BlockDesc(n, h_in, w_in, c_in, c_in, c_in, 1, s * stride, _lib.LASNET_BF16)
        self.wt = _lib.BlockWeights(*(self.wts[k].data_ptr() for k in ("w1", "b1", "w2", "b2", "w3", "b3", "wd", "bd")))
        lib = _lib.load()
        gh, gw = grid(self.h, self.w, s)
        self.ncells = n * gh * gw
        self.mask_buf = torch.empty((n, gh, gw), dtype=torch.uint8, device=device)
        self.logits = torch.empty((n, gh, gw), dtype=torch.float64, device=device)
        self.idx = torch.empty(max(self.ncells, 1), dtype=torch.int32, device=device)
        self.count = torch.zeros(1, dtype=torch.int32, device=device)
        self.ws = torch.zeros(max(lib.lasnet_block_forward_workspace_bytes(ctypes.byref(self.desc), SCHED_SEPARATE), 1),
                              dtype=torch.uint8, device=device)
        self.y = torch.empty((n, self.h, self.w, c_out), dtype=torch.bfloat16, device=device)

    def forward(self, x):
        _lib.check("lasnet_block_forward", _lib.load().lasnet_block_forward(
            ctypes.byref(self.desc), ctypes.byref(self.wt), _p(x), _p(self.y), _p(self.wm), self.bm, SCHED_SEPARATE,
            _p(self.mask_buf), _p(self.idx), _p(self.count), _p(self.ws), self.ws.numel(), _stream()))
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
