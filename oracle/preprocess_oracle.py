"""CPU restatement of the reference's canvas preprocessing (TEST
INFRASTRUCTURE: the checker for the GPU kernel, never a product path).

Follows /root/reference/pkg/src/spikedigits/preprocess.py:
  binarize            :31-35   pixel >= threshold
  crop_to_ink         :38-45   tight half-open bounding box
  resize_preserving_aspect :48-63  longer side -> 20 px, shorter rounded
  center_by_mass      :66-90   centroid to (27/2, 27/2), nearest offset, clamped
  _gaussian_kernel_3x3/blur :93-107  normalised 3x3 Gaussian, sigma 0.8, rint
  preprocess_pipeline :110-115

The resize is Pillow's Image.resize(..., Image.Resampling.BILINEAR) on an
8-bit image (a pinned dependency of the reference: Pillow 12.2 here).  Its
published algorithm (libImaging/Resample.c) is restated, not called:
separable passes (horizontal, then vertical; a pass is skipped when that
dimension keeps its size), each output index xx takes the taps
  center = (xx + 0.5) * scale,  scale = in / out,  support = max(scale, 1)
  xmin = max(int(center - support + 0.5), 0),  xmax = min(int(center + support + 0.5), in)
  w(x) = triangle((x + xmin - center + 0.5) / max(scale, 1)), normalised to sum 1,
converted to fixed point with 22 fractional bits (round half away from
zero), and each output byte is clip8((2^21 + sum in[x] * k[x]) >> 22).
Parity is pinned against the reference's own outputs on 500 synthetic
canvases (tests/golden/canvases.npz, oracle/gen_canvases.py).
"""
from __future__ import annotations

import math

import numpy as np

OUT_SIDE = 28
CONTENT_SIDE = 20
BLUR_SIGMA = 0.8
PRECISION_BITS = 32 - 8 - 2


class BlankDrawing(ValueError):
    pass


def blur_kernel(sigma: float = BLUR_SIGMA) -> np.ndarray:
    """preprocess.py:93-96, the same numpy expression."""
    offsets = np.array([-1.0, 0.0, 1.0])
    gauss = np.exp(-(offsets[:, None] ** 2 + offsets[None, :] ** 2) / (2 * sigma**2))
    return gauss / gauss.sum()


def resize_coeffs(in_size: int, out_size: int):
    """Resample.c precompute_coeffs + normalize_coeffs_8bpc for the bilinear filter."""
    scale = in_size / out_size
    filterscale = max(scale, 1.0)
    support = 1.0 * filterscale
    ss = 1.0 / filterscale
    bounds, coeffs = [], []
    for xx in range(out_size):
        center = (xx + 0.5) * scale
        xmin = max(int(center - support + 0.5), 0)
        xmax = min(int(center + support + 0.5), in_size) - xmin
        k = []
        ww = 0.0
        for x in range(xmax):
            t = abs((x + xmin - center + 0.5) * ss)
            w = 1.0 - t if t < 1.0 else 0.0
            k.append(w)
            ww += w
        if ww != 0.0:
            k = [w / ww for w in k]
        kk = [int(-0.5 + w * (1 << PRECISION_BITS)) if w < 0 else int(0.5 + w * (1 << PRECISION_BITS)) for w in k]
        bounds.append((xmin, xmax))
        coeffs.append(kk)
    return bounds, coeffs


def _pass(img: np.ndarray, out_size: int, axis: int) -> np.ndarray:
    """One 8-bit resampling pass along `axis` (1 = horizontal, 0 = vertical)."""
    a = img if axis == 1 else img.T
    bounds, coeffs = resize_coeffs(a.shape[1], out_size)
    out = np.zeros((a.shape[0], out_size), dtype=np.uint8)
    for xx, ((xmin, xmax), kk) in enumerate(zip(bounds, coeffs)):
        acc = np.full(a.shape[0], 1 << (PRECISION_BITS - 1), dtype=np.int64)
        for x in range(xmax):
            acc += a[:, xmin + x].astype(np.int64) * kk[x]
        out[:, xx] = np.clip(acc >> PRECISION_BITS, 0, 255)
    return out if axis == 1 else out.T


def resize_bilinear(img: np.ndarray, new_w: int, new_h: int) -> np.ndarray:
    """Image.fromarray(img).resize((new_w, new_h), BILINEAR) for uint8 img."""
    out = np.asarray(img, dtype=np.uint8)
    if new_w != out.shape[1]:
        out = _pass(out, new_w, 1)
    if new_h != out.shape[0]:
        out = _pass(out, new_h, 0)
    return np.ascontiguousarray(out)


def preprocess_pil(canvas, threshold: int = 128) -> np.ndarray:
    """The reference's own code path (Pillow's C resize): the CPU baseline
    bench.py times.  Same outputs as preprocess()."""
    from PIL import Image
    return preprocess(canvas, threshold,
                      resize=lambda img, w, h: np.asarray(Image.fromarray(img).resize((w, h), Image.Resampling.BILINEAR),
                                                          dtype=np.uint8))


def preprocess(canvas, threshold: int = 128, resize=None) -> np.ndarray:
    """preprocess_pipeline (preprocess.py:110-115) -> uint8 [28, 28]."""
    arr = np.asarray(canvas)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"canvas must be a 2-D grayscale array, got shape {arr.shape}")
    if not 0 <= threshold <= 255:
        raise ValueError("threshold must lie in 0..255")
    mask = arr >= threshold
    rows = np.flatnonzero(mask.any(axis=1))
    cols = np.flatnonzero(mask.any(axis=0))
    if rows.size == 0:
        raise BlankDrawing("blank drawing: no ink above threshold")
    r0, r1, c0, c1 = int(rows[0]), int(rows[-1]) + 1, int(cols[0]), int(cols[-1]) + 1
    ink = np.where(mask[r0:r1, c0:c1], 255, 0).astype(np.uint8)
    h, w = ink.shape
    if h >= w:
        new_h, new_w = CONTENT_SIDE, max(1, int(math.floor(w * CONTENT_SIDE / h + 0.5)))
    else:
        new_w, new_h = CONTENT_SIDE, max(1, int(math.floor(h * CONTENT_SIDE / w + 0.5)))
    img = (resize or resize_bilinear)(ink, new_w, new_h)
    a = img.astype(np.float64)
    h, w = a.shape
    total = a.sum()
    if total == 0:
        raise BlankDrawing("blank drawing: no mass to center")
    r_bar = float((a.sum(axis=1) * np.arange(h)).sum() / total)
    c_bar = float((a.sum(axis=0) * np.arange(w)).sum() / total)
    center = (OUT_SIDE - 1) / 2.0
    dr = min(max(int(math.floor(center - r_bar + 0.5)), 0), OUT_SIDE - h)
    dc = min(max(int(math.floor(center - c_bar + 0.5)), 0), OUT_SIDE - w)
    placed = np.zeros((OUT_SIDE, OUT_SIDE), dtype=np.uint8)
    placed[dr:dr + h, dc:dc + w] = img
    x = placed.astype(np.float64)
    k = blur_kernel()
    padded = np.pad(x, 1, mode="constant")
    out = np.zeros_like(x)
    for i in range(3):
        for j in range(3):
            out += k[i, j] * padded[i:i + OUT_SIDE, j:j + OUT_SIDE]
    return np.clip(np.rint(out), 0, 255).astype(np.uint8)
