"""Fixtures at the paper's dt = 0.1 ms (N = 1,000), generated FROM THE
REFERENCE (run in the build container):

    python oracle/gen_dt01.py  ->  tests/golden/dt01_reference.npz

* counts of the first 200 config-3 images under W_fix (the reference's own
  batch_counts, one worker per core);
* 40 images of online NormAD from zero weights in config-2 order (the
  reference's train_epoch): per-image counts and the final weights.
"""
from __future__ import annotations

import dataclasses
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "dt01_reference.npz")


def main():
    sys.path.insert(0, REF)
    from spikedigits.evaluate import batch_counts
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import NetworkConfig, run_presentation, zero_weights
    from spikedigits.normad import LearnConfig, train_presentation

    d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
    w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
    bank = default_filter_bank()
    cfg = dataclasses.replace(NetworkConfig(), dt=1e-4)
    t0 = time.time()
    c3 = batch_counts(d["c3_images"][:200], w, bank, cfg, workers=os.cpu_count() or 8)
    order = d["c2_order"][:40]
    wt = zero_weights()
    tc = []
    for i in order:
        wt, cnt = train_presentation(d["c2_images"][i], int(d["c2_labels"][i]), wt, bank, cfg, LearnConfig())
        tc.append(cnt)
    np.savez_compressed(OUT, c3_counts_200=c3.astype(np.int16), train_counts_40=np.stack(tc).astype(np.int16),
                        train_w_40=wt)
    print(f"{time.time() - t0:.0f} s ->", OUT)


if __name__ == "__main__":
    main()
