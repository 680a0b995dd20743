"""Fixtures for the GPU mirrors of two reference tests, generated FROM THE
REFERENCE (run in the build container, where /root/reference exists):

    python oracle/gen_toy.py   ->  tests/golden/toy_reference.npz

* test_normad.py:236-247 (TestConvergence.test_two_class_toy_reaches_perfect_accuracy):
  the 20-image two-class corpus of conftest.py:26-30 (synthetic_dataset(10,
  seed=42), labels 0 and 1), 5 epochs of train_epoch in epoch_permutation(0,
  epoch, 20) order from zero weights; the reference's per-epoch error counts
  and final weights.
* test_network.py:244-258 (test_lateral_inhibition_never_helps_non_winners):
  synthetic_dataset(2, seed=77), weights uniform(0,1)*5e-11 from
  default_rng(99) scaled by 0.5 + l/9; the reference's counts with and
  without lateral inhibition.
"""
from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "toy_reference.npz")


def main():
    sys.path.insert(0, REF)
    from spikedigits.estimator import epoch_permutation
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import N_HIDDEN, N_OUTPUTS, NetworkConfig, run_presentation, zero_weights
    from spikedigits.normad import LearnConfig, train_epoch
    from spikedigits.strokes import synthetic_dataset

    bank, cfg, learn = default_filter_bank(), NetworkConfig(), LearnConfig()
    images, labels = synthetic_dataset(10, seed=42)
    keep = np.isin(labels, [0, 1])
    toy_img, toy_lab = images[keep][:20], labels[keep][:20]
    w = zero_weights()
    orders, errors = [], []
    for epoch in range(5):
        order = epoch_permutation(0, epoch, len(toy_img))
        w, stats = train_epoch(toy_img[order], toy_lab[order], w, bank, cfg, learn)
        orders.append(order)
        errors.append(stats.n_errors)
    inh_img, _ = synthetic_dataset(2, seed=77)
    rng = np.random.default_rng(99)
    inh_w = rng.uniform(0, 1, size=(N_HIDDEN, N_OUTPUTS)) * 5e-11
    inh_w *= 0.5 + np.arange(N_OUTPUTS) / 9.0
    no_inh = dataclasses.replace(cfg, inhibition_weight=0.0)
    with_c = np.stack([run_presentation(im, inh_w, bank, cfg) for im in inh_img])
    without_c = np.stack([run_presentation(im, inh_w, bank, no_inh) for im in inh_img])
    np.savez_compressed(OUT, toy_images=toy_img.astype(np.uint8), toy_labels=toy_lab.astype(np.int64),
                        toy_orders=np.stack(orders), toy_errors=np.array(errors), toy_w=w,
                        inh_images=inh_img.astype(np.uint8), inh_w=inh_w, inh_with=with_c, inh_without=without_c)
    print("errors per epoch", errors, "->", OUT)


if __name__ == "__main__":
    main()
