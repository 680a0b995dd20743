"""Reference counts for all 10,000 images of SURVEY 8(d) config 3
(synthetic_dataset(1000, seed=2000) under W_fix) and all 500 preprocessed
canvases of config 4 at T = 75 ms, generated FROM THE REFERENCE's own
batch_counts (evaluate.py:27-40, one worker process per core):

    python oracle/gen_c3_counts.py  ->  tests/golden/c3_counts_reference.npz
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "c3_counts_reference.npz")


def main():
    sys.path.insert(0, REF)
    from spikedigits.evaluate import batch_counts
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import NetworkConfig

    d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
    w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
    t0 = time.time()
    counts = batch_counts(d["c3_images"], w, default_filter_bank(), NetworkConfig(), workers=os.cpu_count() or 8)
    import dataclasses
    c4 = batch_counts(d["c4_images"], w, default_filter_bank(), dataclasses.replace(NetworkConfig(), t=0.075),
                      workers=os.cpu_count() or 8)
    np.savez_compressed(OUT, counts=counts.astype(np.int16), c4_counts_t75=c4.astype(np.int16))
    print(counts.shape, f"{time.time() - t0:.0f} s ->", OUT)


if __name__ == "__main__":
    main()
