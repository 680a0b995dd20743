"""Generate the config-5 workload and its reference goldens FROM THE REFERENCE.

SURVEY.md 8(d) config 5 (BASELINE.json configs[4]): one full NormAD training
pass over synthetic_dataset(6000, seed=4000) (60,000 images, in
epoch_permutation(0, 0, 60000) order, from zero_weights) followed by
evaluation of synthetic_dataset(1000, seed=5000) (10,000 images).

Run in the build container (where /root/reference exists):

    python oracle/gen_c5.py            # ~35 min: the reference trains 60k images on one core

Writes data/c5_workload.npz (images, labels, order) and
tests/golden/c5_reference.npz (the reference's weights after 1,000 / 10,000 /
60,000 images, its per-image pre-update counts for the whole epoch, and its
eval counts for the first 500 eval images under the final weights).  The GPU
box only reads these fixtures.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    sys.path.insert(0, REF)
    from spikedigits.estimator import epoch_permutation
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import NetworkConfig, run_presentation, zero_weights
    from spikedigits.normad import LearnConfig, train_presentation
    from spikedigits.strokes import synthetic_dataset

    t0 = time.time()
    tr_img, tr_lab = synthetic_dataset(6000, seed=4000)
    ev_img, ev_lab = synthetic_dataset(1000, seed=5000)
    order = epoch_permutation(0, 0, len(tr_img))
    np.savez_compressed(os.path.join(ROOT, "data", "c5_workload.npz"), train_images=tr_img,
                        train_labels=tr_lab, order=order, eval_images=ev_img, eval_labels=ev_lab)
    print(f"workload {time.time() - t0:.1f}s", flush=True)

    bank, cfg, learn = default_filter_bank(), NetworkConfig(), LearnConfig()
    w = zero_weights()
    counts = np.zeros((len(order), 10), dtype=np.int64)
    snaps = {}
    t1 = time.time()
    for i, j in enumerate(order):
        w, counts[i] = train_presentation(tr_img[j], int(tr_lab[j]), w, bank, cfg, learn)
        if i + 1 in (1000, 10000, 60000):
            snaps[f"w_after_{i + 1}"] = w.copy()
            print(f"  {i + 1} images, {time.time() - t1:.0f}s", flush=True)
    train_s = time.time() - t1
    t2 = time.time()
    ev_counts = np.stack([run_presentation(x, w, bank, cfg) for x in ev_img[:500]])
    eval_ms = (time.time() - t2) * 1e3 / 500
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c5_reference.npz"), train_counts=counts,
                        eval_counts_500=ev_counts, train_seconds=train_s, eval_ms_per_img=eval_ms, **snaps)
    print(f"done in {time.time() - t0:.1f}s (train {train_s:.0f}s)")


if __name__ == "__main__":
    main()
