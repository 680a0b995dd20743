"""The reference's hot-path API, executed on the GPU.

Drop-in replacements (paths relative to /root/reference/pkg/src/spikedigits):

  run_presentation   network.py:267-326
  forward_pass       network.py:329-346
  batch_counts       evaluate.py:27-40
  evaluate_dataset   evaluate.py:69-94   (caller of batch_counts)
  train_presentation normad.py:141-162
  train_epoch        normad.py:179-207

Same signatures, return types and exceptions.  Weights arrive and leave as
float64; everything in between runs in the CUDA kernels of libsnn_b200.so.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native
from .engine import get_engine, make_consts
from .params import (N_HIDDEN, N_OUTPUTS, EpochStats, NumericFailureError, SpikeRecord,
                     TAU_SYN_FAST, TAU_SYN_SLOW, as_pixel_batch, as_pixel_image, check_weights,
                     classify)

# shim.install() swaps these for the reference's classes so that callers
# catching spikedigits.normad.NumericFailureError keep working.
_NUMERIC_ERROR = NumericFailureError
_SPIKE_RECORD = SpikeRecord
_EPOCH_STATS = EpochStats


def _torch():
    import torch
    return torch


def _weights(weights) -> np.ndarray:
    w = check_weights(weights)
    if w.shape != (N_HIDDEN, N_OUTPUTS):
        raise ValueError(f"expected weights of shape {(N_HIDDEN, N_OUTPUTS)}, got {w.shape}")
    return np.ascontiguousarray(w)


def _to_device(eng, arr: np.ndarray):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.numel() * t.element_size() >= (1 << 16):
        t = t.pin_memory()
    with torch.cuda.stream(eng.stream):
        return t.to(eng.device, non_blocking=True)


def _fetch(eng, t, dtype=None) -> np.ndarray:
    """Device tensor -> a fresh host array (converted to dtype if given),
    through the engine's pinned staging buffer: one DMA on the engine stream,
    no pageable bounce.  The caller holds eng.lock (the buffer is shared)."""
    import torch
    nb = t.numel() * t.element_size()
    buf = eng.pinned("fetch", nb)
    host = buf[:nb].view(t.dtype).view(t.shape)
    with torch.cuda.stream(eng.stream):
        host.copy_(t, non_blocking=True)
    eng.stream.synchronize()
    a = host.numpy()
    return a.astype(dtype) if dtype is not None else a.copy()


def decode_hidden(raster: np.ndarray, tile_base: int, tile_pos: np.ndarray, n_tiles: int,
                  n_steps: int) -> np.ndarray:
    """Compact raster block of one image -> (N, 8112) bool hidden spike raster.
    Layout (include/snn_b200.h): C = ceil(N/8) chunks, bytes
    [tile_base*C*512 ...), [chunk][tile][half][lane][8 steps], 6-bit masks of
    features half*6 .. half*6+5 of the lane's window."""
    out = np.zeros((n_steps, N_HIDDEN), dtype=bool)
    if n_tiles == 0:
        return out
    nch = -(-n_steps // 8)
    blk = raster[tile_base * nch * 512:(tile_base + n_tiles) * nch * 512]
    blk = blk.reshape(nch, n_tiles, 2, 32, 8).astype(np.int64)
    blk = blk.transpose(0, 4, 1, 2, 3).reshape(nch * 8, n_tiles, 2, 32)[:n_steps]
    masks = blk[:, :, 0, :] | (blk[:, :, 1, :] << 6)              # (N, t, 32) 12-bit
    pos = tile_pos[:n_tiles].astype(np.int64) & 0xFFFF            # (t, 32)
    valid = pos != 0xFFFF
    bits = (masks[..., None] >> np.arange(12)) & 1                 # (N, t, 32, 12)
    idx = pos[:, :, None] * 12 + np.arange(12)                     # (t, 32, 12)
    out[:, idx[valid].ravel()] = bits[:, valid].reshape(n_steps, -1).astype(bool)
    return out


def _replay_hook(on_step: Callable, hidden: np.ndarray, out_mask: np.ndarray, dt: float):
    """Call on_step(n, c_hidden, o_spiked) after the trial, rebuilding c_hidden
    from the recorded hidden spikes with the reference's kernel recursion
    (neurons.py:169-171).  The hook cannot influence the simulation."""
    lam1, lam2 = math.exp(-dt / TAU_SYN_SLOW), math.exp(-dt / TAU_SYN_FAST)
    a = np.zeros(N_HIDDEN)
    b = np.zeros(N_HIDDEN)
    for n in range(hidden.shape[0]):
        bump = hidden[n].astype(np.float64)
        a = a * lam1 + bump
        b = b * lam2 + bump
        on_step(n, a - b, out_mask[n].copy())


_CONSTS_CACHE: dict = {}


def _consts_cached(cfg, filters):
    """make_consts for the serving path, cached on (config, filter taps)."""
    try:
        key = (cfg, np.asarray(filters.weighted, dtype=np.float64).tobytes())
        hit = _CONSTS_CACHE.get(key)
    except TypeError:  # unhashable config object
        return make_consts(cfg, filters)
    if hit is None:
        if len(_CONSTS_CACHE) > 64:
            _CONSTS_CACHE.clear()
        hit = _CONSTS_CACHE[key] = make_consts(cfg, filters)
    return hit


def run_presentation(image, weights, filters, cfg,
                     on_step: Optional[Callable[[int, np.ndarray, np.ndarray], None]] = None,
                     _record_into: Optional[dict] = None) -> np.ndarray:
    """Simulate one image for T/dt steps on the GPU; returns int64[10] counts."""
    eng = get_engine()
    record = on_step is not None or _record_into is not None
    if not record:  # the serving path: cached device weights, one CUDA-graph launch
        with eng.lock:
            eng.weights(weights, check=_weights)  # validated first, as network.py:280 does
            img = as_pixel_image(image)
            return eng.infer_one(_consts_cached(cfg, filters), img)
    w = _weights(weights)
    img = as_pixel_image(image)
    c = _consts_cached(cfg, filters)
    with eng.lock:
        d_img = _to_device(eng, img.reshape(1, -1))
        d_w = _to_device(eng, w)
        out = eng.infer(c, d_img, d_w, raster=record)
        counts = _fetch(eng, out["counts"][0], np.int64)
        if record:
            raster = out["raster"].cpu().numpy()
            tpos = out["tile_pos"][0].cpu().numpy()
            nt = int(out["n_tiles"][0].item())
            tb = int(out["tile_base"][0].item())
            orast = out["out_raster"][0].cpu().numpy().astype(np.int64) & 0x3FF
    if record:
        hidden = decode_hidden(raster, tb, tpos, nt, c.n_steps)
        out_mask = ((orast[:, None] >> np.arange(N_OUTPUTS)) & 1).astype(bool)
        if _record_into is not None:
            _record_into["hidden_mask"] = hidden
            _record_into["output_lists"] = [np.flatnonzero(out_mask[:, l]).tolist() for l in range(N_OUTPUTS)]
        if on_step is not None:
            _replay_hook(on_step, hidden, out_mask, c.dt)
    return counts


def forward_pass(image, weights, filters, cfg):
    """Simulate one presentation and collect the full SpikeRecord."""
    levels = as_pixel_image(image)
    scratch: dict = {}
    counts = run_presentation(levels, weights, filters, cfg, _record_into=scratch)
    eng = get_engine()
    c = make_consts(cfg, filters)
    with eng.lock:
        _, spk = eng.table(c)
        spk = _fetch(eng, spk, bool)
    per_level = [np.flatnonzero(spk[:, k]).tolist() for k in range(256)]
    return _SPIKE_RECORD(
        input_spikes=[list(per_level[k]) for k in levels.ravel()],
        hidden_spikes=[np.flatnonzero(col).tolist() for col in scratch["hidden_mask"].T],
        output_spikes=scratch["output_lists"],
        output_counts=counts,
    )


def batch_counts_device(images_dev, w_dev, c, eng=None):
    """Device-resident batch inference: uint8 [n,784] + f64 [8112,10] device
    tensors -> int32 [n,10] device tensor (no host traffic)."""
    eng = eng or get_engine()
    return eng.infer(c, images_dev, w_dev)["counts"]


def batch_counts(images, weights, filters, cfg, workers: int = 1) -> np.ndarray:
    """Output spike counts per image, (n, 10) int64.  ``workers`` is accepted
    for API compatibility; the batch is data-parallel on the GPU already."""
    imgs = as_pixel_batch(images)
    if len(imgs) == 0:
        return np.zeros((0, N_OUTPUTS), dtype=np.int64)
    c = _consts_cached(cfg, filters)
    eng = get_engine()
    with eng.lock:
        d_w = eng.weights(weights, check=_weights)   # validated once per distinct W, kept on the device
        d_img = eng.upload("images", imgs).view(len(imgs), -1)
        counts = eng.infer(c, d_img, d_w)["counts"]
        return _fetch(eng, counts, np.int64)


@dataclass
class EvalReport:
    n_images: int
    n_correct: int
    confusion: np.ndarray
    mean_image_ms: float
    no_spike_count: int
    t_ms: float = 0.0
    dt_ms: float = 0.0

    @property
    def accuracy(self) -> float:
        return self.n_correct / self.n_images if self.n_images else 0.0

    def to_dict(self) -> dict:
        return {"t_ms": self.t_ms, "dt_ms": self.dt_ms, "n_images": self.n_images,
                "accuracy": self.accuracy, "confusion": self.confusion.tolist(),
                "mean_image_ms": self.mean_image_ms, "no_spike": self.no_spike_count}


def evaluate_dataset(images, labels, weights, filters, cfg, workers: int = 1) -> EvalReport:
    imgs = as_pixel_batch(images)
    labels = np.asarray(labels)
    t0 = time.perf_counter()
    counts = batch_counts(imgs, weights, filters, cfg, workers=workers)
    ms = (time.perf_counter() - t0) * 1e3
    pred = np.argmax(counts, axis=1) if len(counts) else np.zeros(0, dtype=np.int64)
    conf = np.zeros((N_OUTPUTS, N_OUTPUTS), dtype=np.int64)
    np.add.at(conf, (labels.astype(np.int64), pred), 1)
    return EvalReport(n_images=len(imgs), n_correct=int((pred == labels).sum()), confusion=conf,
                      mean_image_ms=ms / len(imgs) if len(imgs) else 0.0,
                      no_spike_count=int((counts.sum(axis=1) == 0).sum()),
                      t_ms=cfg.t * 1e3, dt_ms=cfg.dt * 1e3)


def _train(imgs: np.ndarray, labels: np.ndarray, w: np.ndarray, filters, cfg, learn):
    c = make_consts(cfg, filters, learn)
    eng = get_engine()
    with eng.lock:
        d_img = _to_device(eng, imgs.reshape(len(imgs), -1))
        d_lab = _to_device(eng, labels.astype(np.uint8))
        d_w = _to_device(eng, w)
        counts, status = eng.train(c, d_img, d_lab, d_w)
        st = _fetch(eng, status)
        if st[0] == _native.SNN_ENONFINITE:
            raise _NUMERIC_ERROR("weight update produced non-finite values")
        if st[0] != 0:
            raise _native.NativeError(int(st[0]), "training kernel failed")
        return d_w.cpu().numpy(), counts.cpu().numpy().astype(np.int64)


def _labels(labels, n: int) -> np.ndarray:
    lab = np.asarray(labels)
    if len(lab) != n:
        raise ValueError("images and labels length mismatch")
    if n and (lab.min() < 0 or lab.max() >= N_OUTPUTS):
        raise ValueError("labels must be digits 0..9")
    return np.array([int(x) for x in lab], dtype=np.int64)


def train_presentation(image, label: int, weights, filters, cfg, learn):
    """One supervised presentation; returns (new float64 weights, int64 counts)."""
    img = as_pixel_image(image)
    lab = int(label)
    if not -N_OUTPUTS <= lab < N_OUTPUTS:   # numpy indexing semantics of normad.py:137
        raise IndexError(f"index {lab} is out of bounds for axis 1 with size {N_OUTPUTS}")
    lab %= N_OUTPUTS
    w, counts = _train(img.reshape(1, 28, 28), np.array([lab]), _weights(weights), filters, cfg, learn)
    return w, counts[0]


def train_epoch(images, labels, weights, filters, cfg, learn):
    """One sequential online NormAD pass in the given order -> (W, EpochStats)."""
    imgs = as_pixel_batch(images)
    lab = _labels(labels, len(imgs))
    stats = _EPOCH_STATS()
    t0 = time.perf_counter()
    w = _weights(weights)
    if len(imgs):
        w, counts = _train(imgs, lab, w, filters, cfg, learn)
        pred = np.argmax(counts, axis=1)
        wrong = pred != lab
        stats.n_images = len(imgs)
        stats.n_errors = int(wrong.sum())
        for l in lab[wrong]:
            stats.error_counts[int(l)] += 1
    else:
        w = np.array(w, copy=True)
    stats.wall_seconds = time.perf_counter() - t0
    return w, stats


__all__ = ["run_presentation", "forward_pass", "batch_counts", "batch_counts_device", "evaluate_dataset",
           "EvalReport", "train_presentation", "train_epoch", "classify", "decode_hidden"]
