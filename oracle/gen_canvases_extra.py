"""Reference outputs for canvases off the uint8 / <=1024 px path, generated
FROM THE REFERENCE's own preprocess_pipeline (preprocess.py:110-115):

    python oracle/gen_canvases_extra.py -> tests/golden/canvases_extra.npz

c0: float64 canvas, threshold 127.5      c1: int16 with values < 0 and > 255, threshold 200
c2: bool canvas, threshold 1             c3: uint8 1500 x 1300, small drawing, threshold 128
c4: uint8 2000 x 1800, drawing 900 px across, threshold 90
c5: float32 1100 x 1030 with a thin stroke, threshold 0.5
Keys: canvas<i>, threshold<i> (float64 scalar), out<i> (uint8 [28, 28]).
Test infrastructure only.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "canvases_extra.npz")


def canvases():
    rng = np.random.default_rng(77)
    yy, xx = np.mgrid[0:96, 0:80]
    blob = np.exp(-((yy - 40.0) ** 2 / 300 + (xx - 35.0) ** 2 / 120)) * 300.0 - 20.0
    c0 = blob.astype(np.float64)
    c1 = (blob + rng.normal(0, 30, blob.shape)).astype(np.int16)
    c2 = blob > 150.0
    c3 = np.zeros((1500, 1300), dtype=np.uint8)
    c3[700:760, 600:612] = 255
    c3[700:712, 600:650] = 220
    c4 = np.zeros((2000, 1800), dtype=np.uint8)
    r = np.arange(2000)[:, None]
    c = np.arange(1800)[None, :]
    ring = np.abs(np.hypot(r - 1000.0, c - 900.0) - 420.0) < 25.0
    c4[ring] = 200
    c4[1000:1010, 450:1350] = 120
    c5 = np.zeros((1100, 1030), dtype=np.float32)
    c5[100:1000, 500:503] = 0.75
    c5[540:545, 40:1000] = 0.5
    return [(c0, 127.5), (c1, 200), (c2, 1), (c3, 128), (c4, 90), (c5, 0.5)]


def main():
    sys.path.insert(0, REF)
    from spikedigits.preprocess import preprocess_pipeline
    z = {}
    for i, (cv, thr) in enumerate(canvases()):
        z[f"canvas{i}"] = cv
        z[f"threshold{i}"] = np.float64(thr)
        z[f"out{i}"] = preprocess_pipeline(cv, thr)
    np.savez_compressed(OUT, **z)
    print(len(z) // 3, "canvases ->", OUT)


if __name__ == "__main__":
    main()
