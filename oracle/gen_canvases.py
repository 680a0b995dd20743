"""Canvas fixtures for the GPU preprocessing, generated FROM THE REFERENCE
(run in the build container, where /root/reference exists):

    python oracle/gen_canvases.py  ->  tests/golden/canvases.npz

* the 500 synthetic user canvases of SURVEY 8(d) config 4
  (strokes.synthetic_canvases(500, seed=3000)) and preprocess_pipeline's
  outputs for them (threshold 128);
* 200 extra canvases exercising the resize paths (non-square, tall, wide,
  tiny ink, canvases smaller than 20 px so the resize upsamples, thresholds
  64 / 200) with the reference's outputs, and blank canvases (the
  reference raises BlankDrawingError: output all 0, flag 1).
Canvases have different shapes: stored flat with per-canvas (h, w, offset).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "canvases.npz")


def main():
    sys.path.insert(0, REF)
    from spikedigits.preprocess import BlankDrawingError, preprocess_pipeline
    from spikedigits.strokes import synthetic_canvases

    canv = [c for c, _ in synthetic_canvases(500, seed=3000)]
    thr = [128] * len(canv)
    rng = np.random.default_rng(7)
    for k in range(200):
        kind = k % 5
        if kind == 0:    # non-square, random strokes
            h, w = int(rng.integers(30, 300)), int(rng.integers(30, 300))
        elif kind == 1:  # tall / wide extremes
            h, w = (int(rng.integers(100, 400)), int(rng.integers(5, 30))) if k % 2 else \
                   (int(rng.integers(5, 30)), int(rng.integers(100, 400)))
        elif kind == 2:  # small canvases: the resize upsamples
            h, w = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        elif kind == 3:  # sparse ink, one or two pixels
            h, w = int(rng.integers(20, 120)), int(rng.integers(20, 120))
        else:            # blank or nearly blank
            h, w = int(rng.integers(10, 80)), int(rng.integers(10, 80))
        c = np.zeros((h, w), dtype=np.uint8)
        if kind in (0, 1, 2):
            n = int(rng.integers(1, 6))
            for _ in range(n):
                r0, r1 = sorted(rng.integers(0, h, 2))
                c0, c1 = sorted(rng.integers(0, w, 2))
                c[r0:r1 + 1, c0:c1 + 1] = rng.integers(0, 256, (r1 - r0 + 1, c1 - c0 + 1))
        elif kind == 3:
            for _ in range(int(rng.integers(1, 3))):
                c[int(rng.integers(0, h)), int(rng.integers(0, w))] = 255
        elif k % 10 == 4:
            c[:] = rng.integers(0, 100, (h, w))  # below every threshold used: blank
        canv.append(c)
        thr.append(int((128, 64, 200)[k % 3]))
    outs, blank = [], []
    for c, t in zip(canv, thr):
        try:
            outs.append(preprocess_pipeline(c, threshold=t))
            blank.append(0)
        except BlankDrawingError:
            outs.append(np.zeros((28, 28), dtype=np.uint8))
            blank.append(1)
    shapes = np.array([c.shape for c in canv], dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(shapes[:, 0] * shapes[:, 1])]).astype(np.int64)
    flat = np.concatenate([c.ravel() for c in canv]).astype(np.uint8)
    np.savez_compressed(OUT, pixels=flat, shapes=shapes, offsets=offs, thresholds=np.array(thr, dtype=np.int64),
                        outputs=np.stack(outs), blank=np.array(blank, dtype=np.int64))
    print(len(canv), "canvases,", int(sum(blank)), "blank ->", OUT, os.path.getsize(OUT) // 1024, "KB")


if __name__ == "__main__":
    main()
