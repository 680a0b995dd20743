"""Device engine: constants, cached input tables, workspaces, stream, lock.

One Engine per CUDA device.  All kernels run on the engine's own stream
through the C ABI (``_native``); torch is used only for device memory and
host<->device copies.  Calls are serialised by a lock, so the FastAPI
thread-pool callers of ``run_presentation`` (service.py:107) are safe.
"""
from __future__ import annotations

import ctypes
import math
import threading
from collections import OrderedDict

import numpy as np

from . import _native
from .params import N_HIDDEN, N_INPUTS, N_OUTPUTS, TAU_LEARN, TAU_SYN_FAST, TAU_SYN_SLOW, desired_period

_ENGINES: dict = {}
_ENGINES_LOCK = threading.Lock()


def _torch():
    import torch
    return torch


def _lif(p, dt: float) -> _native.LifC:
    """neurons.py:109-118, same float expression order as the reference."""
    g, cap = float(p.leak_conductance), float(p.capacitance)
    beta = dt * (2.0 - g * dt / cap) / (2.0 * cap)
    return _native.LifC(g, float(p.rest_potential), float(p.threshold), beta, float(p.refractory) / dt)


def make_consts(cfg, filters, learn=None) -> _native.ConstsC:
    """Flatten NetworkConfig/FilterBank/LearnConfig (reference or mirror objects)."""
    dt = float(cfg.dt)
    c = _native.ConstsC()
    c.n_steps = int(round(float(cfg.t) / dt))
    c.desired_period = desired_period(float(cfg.t), dt, float(cfg.desired_rate))
    c.dt = dt
    c.i0 = float(cfg.encoding.i_0)
    c.ip = float(cfg.encoding.i_p)
    c.lif_in = _lif(cfg.input_lif, dt)
    c.lif_hid = _lif(cfg.hidden_lif, dt)
    c.lif_out = _lif(cfg.output_lif, dt)
    c.decay_slow = math.exp(-dt / TAU_SYN_SLOW)      # neurons.py:148-150
    c.decay_fast = math.exp(-dt / TAU_SYN_FAST)
    c.decay_learn = math.exp(-dt / TAU_LEARN)        # normad.py:82
    c.dhat_scale = dt / float(cfg.output_lif.capacitance)   # normad.py:83
    c.inhibition = float(cfg.inhibition_weight)
    if learn is not None:
        c.learning_rate = float(learn.learning_rate)
        c.norm_eps = float(learn.norm_epsilon)
    taps = np.ascontiguousarray(np.asarray(filters.weighted, dtype=np.float64).reshape(12, 9))
    ctypes.memmove(ctypes.addressof(c.taps), taps.ctypes.data, taps.nbytes)
    # network.py:284-285 raises on non-finite hidden currents.  |c_in| <= 1/(1-decay_slow),
    # so finite currents are guaranteed unless the gains are astronomically large.
    bound = 9.0 * float(np.max(np.abs(taps))) / (1.0 - c.decay_slow)
    if not (bound < 1e300):
        raise ValueError("hidden currents contain non-finite values")
    return c


def table_key(c: _native.ConstsC):
    li = c.lif_in
    return (c.n_steps, c.dt, c.i0, c.ip, li.g, li.el, li.vt, li.beta, li.refr, c.decay_slow, c.decay_fast)


MAX_TABLES = 8
MAX_GRAPHS = 16


class Engine:
    def __init__(self, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1711_03637_b200 needs a CUDA device (no CPU fallback)")
        self.lib = _native.load()
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
        self.lock = threading.RLock()
        self._tables: OrderedDict = OrderedDict()   # LRU, MAX_TABLES entries
        self._ws: dict = {}
        self._w_host = None      # host copy of the weights last uploaded by weights()
        self._w_dev = None
        # batch-1 CUDA graphs per configuration (infer_one), LRU of MAX_GRAPHS;
        # each entry holds every device buffer its graph reads (table, image,
        # counts, workspace), so a graph never outlives the memory it captured
        self._graphs: OrderedDict = OrderedDict()
        self._pinned: dict = {}   # grow-only pinned host staging buffers

    # ------------------------------------------------------------ helpers
    @property
    def sptr(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def buffer(self, name: str, nbytes: int):
        """Grow-only scratch buffer (uint8 tensor) on this device."""
        torch = _torch()
        buf = self._ws.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[name] = buf
        return buf

    def pinned(self, name: str, nbytes: int):
        """Grow-only pinned host staging buffer (uint8 tensor)."""
        torch = _torch()
        buf = self._pinned.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 4096), dtype=torch.uint8).pin_memory()
            self._pinned[name] = buf
        return buf

    def upload(self, name: str, arr: np.ndarray):
        """Host array -> device uint8 tensor of the same bytes (grow-only
        device buffer `name`), copied straight from the caller's pageable
        memory on the engine's stream: the driver stages and DMAs it in
        pipelined chunks, measured faster on B200 hosts than a host copy into
        pinned memory followed by a pinned H2D (0.39 vs 0.39 + 0.34 ms for
        7.8 MB, scripts/e2e_breakdown.py).  The caller holds the lock."""
        torch = _torch()
        src = np.ascontiguousarray(arr).reshape(-1).view(np.uint8)
        nb = int(src.nbytes)
        dev = self.buffer(name, nb)
        with torch.cuda.stream(self.stream):
            dev[:nb].copy_(torch.from_numpy(src), non_blocking=True)
        return dev[:nb]

    def table(self, c: _native.ConstsC):
        """(c_table [N,256] f64, spike table [N,256] u8) on device, cached per config."""
        torch = _torch()
        key = table_key(c)
        hit = self._tables.get(key)
        if hit is not None:
            self._tables.move_to_end(key)
        else:
            with torch.cuda.stream(self.stream):
                ctab = torch.empty((c.n_steps, 256), dtype=torch.float64, device=self.device)
                spk = torch.empty((c.n_steps, 256), dtype=torch.uint8, device=self.device)
            _native.check(self.lib.snn_input_table(ctypes.byref(c), ctab.data_ptr(), spk.data_ptr(), self.sptr))
            torch.cuda.current_stream(self.device).wait_stream(self.stream)
            if len(self._tables) >= MAX_TABLES:
                self._tables.popitem(last=False)   # graphs keep their own reference to it
            hit = self._tables[key] = (ctab, spk)
        return hit

    # ------------------------------------------------------------ inference
    def infer(self, c, images, w, *, raster=False, trace=False, ties=False, max_chunk=None):
        """Run n presentations.  images: uint8 [n,784] device tensor; w: f64
        [8112,10] device tensor.  Returns dict of device tensors (counts int32
        [n,10]; optionally raster/tile_pos/n_tiles/tile_base/out_raster,
        ff/v_out/v_hid, near_ties int32 [n] (snn_infer_out_t.near_ties))."""
        torch = _torch()
        n = int(images.shape[0])
        N = c.n_steps
        ctab, _ = self.table(c)
        dev = self.device
        self.stream.wait_stream(torch.cuda.current_stream(dev))   # inputs made on the caller's stream
        with torch.cuda.stream(self.stream):
            out = {"counts": torch.empty((n, N_OUTPUTS), dtype=torch.int32, device=dev)}
            if raster:  # compact layout, see include/snn_b200.h
                out["raster"] = torch.empty((_native.raster_bytes(n, N),), dtype=torch.uint8, device=dev)
                out["tile_pos"] = torch.empty((n, _native.MAX_TILES, _native.TILE), dtype=torch.int16, device=dev)
                out["n_tiles"] = torch.empty((n,), dtype=torch.int32, device=dev)
                out["tile_base"] = torch.empty((n + 1,), dtype=torch.int32, device=dev)
                out["out_raster"] = torch.empty((n, N), dtype=torch.int16, device=dev)
            if ties:
                out["near_ties"] = torch.empty((n,), dtype=torch.int32, device=dev)
            out["hidden_redo"] = torch.zeros((1,), dtype=torch.int32, device=dev)
            if trace:
                out["ff"] = torch.empty((n, N, N_OUTPUTS), dtype=torch.float64, device=dev)
                out["v_out"] = torch.empty((n, N, N_OUTPUTS), dtype=torch.float64, device=dev)
                out["v_hid"] = torch.full((n, N, N_HIDDEN), float(c.lif_hid.el), dtype=torch.float64, device=dev)
        per_img = max(1, self.lib.snn_infer_workspace(ctypes.byref(c), 1))
        chunk = max(1, min(n, (4 << 30) // per_img))
        if max_chunk:
            chunk = min(chunk, max_chunk)
        if raster:
            chunk = n  # the compact raster of one call is indexed by one tile_base
        assert images.dtype == torch.uint8 and images.is_contiguous() and images.shape[1] == N_INPUTS
        assert w.dtype == torch.float64 and w.is_contiguous() and tuple(w.shape) == (N_HIDDEN, N_OUTPUTS)
        for i0 in range(0, n, chunk):
            cn = min(chunk, n - i0)
            ws_bytes = self.lib.snn_infer_workspace(ctypes.byref(c), cn)
            ws = self.buffer("infer", ws_bytes)
            o = _native.InferOutC()
            for name, t in out.items():
                whole = name in ("raster", "tile_base", "hidden_redo")
                setattr(o, name, t.data_ptr() if whole else t[i0:i0 + cn].data_ptr())
            _native.check(self.lib.snn_infer(
                ctypes.byref(c), images[i0:i0 + cn].data_ptr(), cn, w.data_ptr(), ctab.data_ptr(),
                ctypes.byref(o), ws.data_ptr(), ws_bytes, self.sptr))
        torch.cuda.current_stream(dev).wait_stream(self.stream)   # results safe on the caller's stream
        return out

    # ------------------------------------------------------------ serving (batch 1)
    def weights(self, w, check=None):
        """Device copy of [8112,10] host weights, re-uploaded only when their
        values change (one compare per call; the serving engine keeps one
        checkpoint for many requests, service.py:54-79).  `check` validates
        and converts a new array (validation.check_weights); an array equal to
        the cached one was validated already.  The device buffer's address
        never changes, so captured graphs stay valid."""
        torch = _torch()
        if self._w_dev is None:
            with torch.cuda.stream(self.stream):
                self._w_dev = torch.empty((N_HIDDEN, N_OUTPUTS), dtype=torch.float64, device=self.device)
        if self._w_host is not None and np.shape(w) == self._w_host.shape and np.array_equal(self._w_host, w):
            return self._w_dev
        host = check(w) if check is not None else np.asarray(w, dtype=np.float64)
        if host.shape != (N_HIDDEN, N_OUTPUTS):
            raise ValueError(f"expected weights of shape {(N_HIDDEN, N_OUTPUTS)}, got {host.shape}")
        self._w_host = np.array(host, dtype=np.float64, copy=True)
        with torch.cuda.stream(self.stream):
            self._w_dev.copy_(torch.from_numpy(self._w_host).pin_memory(), non_blocking=True)
        return self._w_dev

    def infer_one(self, c, image: np.ndarray, w=None, check=None) -> np.ndarray:
        """One presentation through a CUDA graph captured per configuration:
        one graph launch holding the pinned H2D of the 784-byte image,
        k_prep .. k_output and the D2H of the counts.  Same kernels and results as infer().
        Without `w`, the weights last set by weights() are used."""
        torch = _torch()
        d_w = self.weights(w, check) if w is not None else self._w_dev
        key = bytes(c)
        gr = self._graphs.get(key)
        if gr is not None:
            self._graphs.move_to_end(key)
        else:
            if len(self._graphs) >= MAX_GRAPHS:
                self._graphs.popitem(last=False)  # drops the graph with its buffers
            ctab, _ = self.table(c)
            with torch.cuda.stream(self.stream):
                img_d = torch.zeros((1, N_INPUTS), dtype=torch.uint8, device=self.device)
                cnt_d = torch.zeros((1, N_OUTPUTS), dtype=torch.int32, device=self.device)
            ws_bytes = self.lib.snn_infer_workspace(ctypes.byref(c), 1)
            with torch.cuda.stream(self.stream):
                ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=self.device)
            o = _native.InferOutC()
            o.counts = cnt_d.data_ptr()
            args = (ctypes.byref(c), img_d.data_ptr(), 1, d_w.data_ptr(), ctab.data_ptr(), ctypes.byref(o),
                    ws.data_ptr(), ws_bytes, self.sptr)
            _native.check(self.lib.snn_infer(*args))   # first launch: lazy attributes, module load
            self.stream.synchronize()
            img_h = torch.zeros((1, N_INPUTS), dtype=torch.uint8).pin_memory()
            cnt_h = torch.zeros((1, N_OUTPUTS), dtype=torch.int32).pin_memory()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):  # the copies are graph nodes too
                img_d.copy_(img_h, non_blocking=True)
                _native.check(self.lib.snn_infer(*args))
                cnt_h.copy_(cnt_d, non_blocking=True)
            gr = self._graphs[key] = {"g": g, "img": img_d, "cnt": cnt_d, "ws": ws, "c": c, "o": o, "ctab": ctab,
                                      "img_h": img_h, "cnt_h": cnt_h,
                                      "img_np": img_h.numpy()[0], "cnt_np": cnt_h.numpy()[0]}
        gr["img_np"][:] = image.reshape(-1)
        with torch.cuda.stream(self.stream):
            gr["g"].replay()
        self.stream.synchronize()
        return gr["cnt_np"].astype(np.int64)

    # ------------------------------------------------------------ training
    def train(self, c, images, labels, w):
        """Sequential NormAD over n images (device tensors), updating w in place.
        Returns (counts int32 [n,10] device, status int32 [4] device)."""
        torch = _torch()
        n = int(images.shape[0])
        assert images.dtype == torch.uint8 and images.is_contiguous() and tuple(images.shape[1:]) == (N_INPUTS,)
        assert labels.dtype == torch.uint8 and labels.is_contiguous() and tuple(labels.shape) == (n,)
        assert w.dtype == torch.float64 and w.is_contiguous() and tuple(w.shape) == (N_HIDDEN, N_OUTPUTS)
        ctab, _ = self.table(c)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            counts = torch.zeros((n, N_OUTPUTS), dtype=torch.int32, device=self.device)
            status = torch.zeros((4,), dtype=torch.int32, device=self.device)
        ws_bytes = self.lib.snn_train_workspace(ctypes.byref(c), n)
        ws = self.buffer("train", ws_bytes)
        _native.check(self.lib.snn_train(
            ctypes.byref(c), images.data_ptr(), labels.data_ptr(), n, w.data_ptr(), ctab.data_ptr(),
            counts.data_ptr(), status.data_ptr(), ws.data_ptr(), ws_bytes, self.sptr))
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return counts, status


def get_engine(device=None) -> Engine:
    torch = _torch()
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1711_03637_b200 needs a CUDA device (no CPU fallback)")
        device = torch.cuda.current_device()
    key = str(torch.device(device) if not isinstance(device, int) else torch.device("cuda", device))
    with _ENGINES_LOCK:
        eng = _ENGINES.get(key)
        if eng is None:
            eng = _ENGINES[key] = Engine(key)
        return eng
