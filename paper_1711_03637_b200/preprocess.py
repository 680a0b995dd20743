"""GPU canvas preprocessing with the reference's API
(/root/reference/pkg/src/spikedigits/preprocess.py:110-115).

``preprocess_pipeline(canvas, threshold=128)`` turns one user-drawn
grayscale canvas into the 28x28 uint8 image the network takes (binarize,
crop to ink, longer side to 20 px with Pillow's BILINEAR resampling, place
by centre of mass, 3x3 Gaussian blur) on the GPU (``k_preprocess`` through
``snn_preprocess``); ``preprocess_batch`` does many canvases in one launch.
Outputs are bit-identical to the reference's; a canvas without ink raises
``BlankDrawingError`` like the reference.

Host-side normalisation, exact by construction (everything after
``binarize`` depends only on the ink mask, preprocess.py:110-115):
* a uint8 canvas with a threshold t goes to the kernel as is with
  ceil(t) (for integer pixels ``x >= t  <=>  x >= ceil(t)``);
* any other dtype (float, int16, bool, ...) is binarized on the host with
  the reference's own comparison ``canvas >= threshold`` and sent as a
  0/255 mask with threshold 128;
* a canvas wider or taller than the kernel's 1024 px is cropped on the host
  to the ink's bounding box first (the reference crops to the same box,
  preprocess.py:38-45, before anything else); only an INK extent beyond
  1024 px per side is rejected (ValueError; the service itself caps canvases
  at 1024 px, service.py:31).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native

OUT_SIDE = 28
CONTENT_SIDE = 20
BLUR_SIGMA = 0.8
MAX_SIDE = 1024


class BlankDrawingError(ValueError):
    """The canvas holds no ink above the binarization threshold."""


def _blur_kernel(sigma: float = BLUR_SIGMA) -> np.ndarray:
    """preprocess.py:93-96, the same numpy expression (passed to the kernel)."""
    offsets = np.array([-1.0, 0.0, 1.0])
    gauss = np.exp(-(offsets[:, None] ** 2 + offsets[None, :] ** 2) / (2 * sigma**2))
    return np.ascontiguousarray(gauss / gauss.sum(), dtype=np.float64)


_BLUR = _blur_kernel()
_BLANK_ERROR = BlankDrawingError  # shim.install() points this at the reference's class


def _as_canvas(canvas) -> np.ndarray:
    arr = np.asarray(canvas)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"canvas must be a 2-D grayscale array, got shape {arr.shape}")
    return arr


def _check_threshold(threshold):
    """preprocess.py:31-35 (binarize): the same test, the same message."""
    if not 0 <= threshold <= 255:
        raise ValueError("threshold must lie in 0..255")
    return threshold


def _prepare(canvas, threshold):
    """(uint8 canvas <= 1024 px per side, int threshold) with the same ink
    mask as ``canvas >= threshold`` (see the module docstring)."""
    arr = _as_canvas(canvas)
    thr = _check_threshold(threshold)
    if arr.dtype == np.uint8:
        t = int(np.ceil(thr))
    else:  # the reference's own comparison, on the host
        arr = np.where(arr >= thr, np.uint8(255), np.uint8(0))
        t = 128
    if arr.shape[0] > MAX_SIDE or arr.shape[1] > MAX_SIDE:
        mask = arr >= t
        rows, cols = np.flatnonzero(mask.any(axis=1)), np.flatnonzero(mask.any(axis=0))
        if rows.size == 0:  # no ink (so t > 0): a 1x1 canvas without ink reports the blank drawing
            arr = np.zeros((1, 1), dtype=np.uint8)
        else:
            arr = arr[rows[0]:rows[-1] + 1, cols[0]:cols[-1] + 1]
        if arr.shape[0] > MAX_SIDE or arr.shape[1] > MAX_SIDE:
            raise ValueError(f"ink extent {arr.shape} exceeds {MAX_SIDE} px per side")
    return np.ascontiguousarray(arr), t


def preprocess_batch(canvases, threshold=128):
    """Preprocess many canvases in one launch.  Returns (images uint8
    [n, 28, 28], blank bool [n]); blank canvases give an all-zero image."""
    from .engine import get_engine, _torch
    canvases = list(canvases)
    n = len(canvases)
    ts = list(np.broadcast_to(np.asarray(threshold, dtype=object), (n,))) if n else []
    prep = [_prepare(c, t) for c, t in zip(canvases, ts)]
    cs = [p[0] for p in prep]
    thr = np.array([p[1] for p in prep], dtype=np.int32)
    if n == 0:
        return np.zeros((0, OUT_SIDE, OUT_SIDE), dtype=np.uint8), np.zeros(0, dtype=bool)
    shapes = np.array([c.shape for c in cs], dtype=np.int32)
    sizes = shapes[:, 0].astype(np.int64) * shapes[:, 1]
    offsets = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    total = int(sizes.sum())
    torch = _torch()
    eng = get_engine()
    with eng.lock:
        # one pinned staging block: pixels | offsets | shapes | thresholds
        nb = [total, 8 * n, 8 * n, 4 * n]
        cuts = np.cumsum([0] + [(b + 15) // 16 * 16 for b in nb])
        host = eng.pinned("pre_in", int(cuts[-1])).numpy()
        host[cuts[0]:cuts[0] + total] = np.concatenate([c.ravel() for c in cs]) if n > 1 else cs[0].ravel()
        host[cuts[1]:cuts[1] + nb[1]] = offsets.view(np.uint8)
        host[cuts[2]:cuts[2] + nb[2]] = shapes.view(np.uint8).reshape(-1)
        host[cuts[3]:cuts[3] + nb[3]] = thr.view(np.uint8)
        dev = eng.buffer("pre_in", int(cuts[-1]))
        out = eng.buffer("pre_out", n * (OUT_SIDE * OUT_SIDE + 4))
        with torch.cuda.stream(eng.stream):
            dev[:int(cuts[-1])].copy_(eng.pinned("pre_in", int(cuts[-1]))[:int(cuts[-1])], non_blocking=True)
        base = dev.data_ptr()
        st_off = n * OUT_SIDE * OUT_SIDE
        _native.check(eng.lib.snn_preprocess(
            ctypes.c_void_p(base + int(cuts[0])), ctypes.c_void_p(base + int(cuts[1])),
            ctypes.c_void_p(base + int(cuts[2])), ctypes.c_void_p(base + int(cuts[3])), n,
            _BLUR.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(out.data_ptr() + st_off), eng.sptr))
        res = eng.pinned("pre_out", n * (OUT_SIDE * OUT_SIDE + 4))
        with torch.cuda.stream(eng.stream):
            res[:n * (OUT_SIDE * OUT_SIDE + 4)].copy_(out[:n * (OUT_SIDE * OUT_SIDE + 4)], non_blocking=True)
        eng.stream.synchronize()
        r = res.numpy()
        images = r[:st_off].reshape(n, OUT_SIDE, OUT_SIDE).copy()
        status = r[st_off:st_off + 4 * n].view(np.int32).copy()
    if (status == 2).any():
        raise ValueError("canvas shape outside 1..1024")
    return images, status == 1


def preprocess_pipeline(canvas, threshold: int = 128) -> np.ndarray:
    """Full canvas-to-28x28 pipeline on the GPU; raises BlankDrawingError on empty ink."""
    images, blank = preprocess_batch([canvas], threshold)
    if blank[0]:
        raise _BLANK_ERROR("blank drawing: no ink above threshold")
    return images[0]


__all__ = ["preprocess_pipeline", "preprocess_batch", "BlankDrawingError"]
