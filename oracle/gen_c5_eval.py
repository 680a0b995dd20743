"""Reference eval counts for ALL 10,000 config-5 eval images, generated FROM
THE REFERENCE's own batch_counts (evaluate.py:27-40, one worker process per
core) under the reference's own weights after the 60,000-image NormAD pass
(tests/golden/c5_reference.npz "w_after_60000", written by gen_c5.py):

    python oracle/gen_c5_eval.py  ->  tests/golden/c5_eval_reference.npz

Test infrastructure only (the GPU box reads the fixture, never the reference).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "c5_eval_reference.npz")


def main():
    sys.path.insert(0, REF)
    from spikedigits.evaluate import batch_counts
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import NetworkConfig

    d5 = np.load(os.path.join(ROOT, "data", "c5_workload.npz"))
    w = np.load(os.path.join(ROOT, "tests", "golden", "c5_reference.npz"))["w_after_60000"]
    t0 = time.time()
    counts = batch_counts(d5["eval_images"], w, default_filter_bank(), NetworkConfig(),
                          workers=os.cpu_count() or 8)
    np.savez_compressed(OUT, eval_counts=counts.astype(np.int16))
    print(counts.shape, f"{time.time() - t0:.0f} s ->", OUT)


if __name__ == "__main__":
    main()
