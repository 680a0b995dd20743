"""Generate the golden fixtures under tests/golden/ and data/ FROM THE REFERENCE.

Run in the build container (where /root/reference exists):

    python oracle/gen_golden.py

Everything here is produced by calling the unmodified reference package
(``/root/reference/pkg/src/spikedigits``) through its public API, so the
committed vectors pin both the oracle (tests/test_oracle_golden.py) and the
GPU path (tests/test_gpu_parity.py) to the reference's own outputs.
The GPU box never reads /root/reference; it only reads these fixtures.

Workloads follow SURVEY.md section 8(d):
  c1  single image             synthetic_dataset(1, seed=1000)[0][0]
  c2  NormAD 1,000             synthetic_dataset(100, seed=1000), epoch_permutation(0,0,1000)
  c3  batched 10,000           synthetic_dataset(1000, seed=2000)
  c4  real-time 500 canvases   synthetic_canvases(500, seed=3000) -> preprocess_pipeline
  W_fix = train_epoch over c2 from zero_weights (one epoch)
"""
from __future__ import annotations

import dataclasses
import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")


def main():
    sys.path.insert(0, REF)
    from spikedigits.estimator import epoch_permutation
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import (NetworkConfig, _input_tables, forward_pass,
                                     hidden_current_series, run_presentation, zero_weights)
    from spikedigits.normad import LearnConfig, train_epoch, train_presentation
    from spikedigits.preprocess import preprocess_pipeline
    from spikedigits.strokes import synthetic_canvases, synthetic_dataset

    os.makedirs(GOLD, exist_ok=True)
    os.makedirs(DATA, exist_ok=True)
    bank = default_filter_bank()
    cfg = NetworkConfig()
    t0 = time.time()

    # ---- workloads (data/) -------------------------------------------------
    c2_img, c2_lab = synthetic_dataset(100, seed=1000)
    order = epoch_permutation(0, 0, len(c2_img))
    c3_img, c3_lab = synthetic_dataset(1000, seed=2000)
    canv = synthetic_canvases(500, seed=3000)
    c4_img = np.stack([preprocess_pipeline(c) for c, _ in canv])
    c4_lab = np.array([d for _, d in canv], dtype=np.uint8)
    print(f"workloads {time.time()-t0:.1f}s", flush=True)

    # ---- W_fix: one reference epoch over c2 (the training trajectory golden) ----
    learn = LearnConfig()
    w = zero_weights()
    snaps = {}
    counts_tr = np.zeros((len(order), 10), dtype=np.int64)
    t1 = time.time()
    for i, j in enumerate(order):
        w, counts_tr[i] = train_presentation(c2_img[j], int(c2_lab[j]), w, bank, cfg, learn)
        if i + 1 in (1, 2, 5, 20, 100):
            snaps[f"w_after_{i+1}"] = w.copy()
    train_s = time.time() - t1
    w_fix = w
    # sanity: identical to train_epoch (the public entry point)
    w_chk, stats = train_epoch(c2_img[order][:20], c2_lab[order][:20], zero_weights(), bank, cfg, learn)
    assert np.array_equal(w_chk, snaps["w_after_20"])
    print(f"train {train_s:.1f}s", flush=True)

    np.savez_compressed(os.path.join(DATA, "workloads.npz"),
                        c2_images=c2_img, c2_labels=c2_lab, c2_order=order,
                        c3_images=c3_img, c3_labels=c3_lab,
                        c4_images=c4_img, c4_labels=c4_lab)
    np.savez_compressed(os.path.join(DATA, "w_fix.npz"), w_fix=w_fix,
                        train_counts=counts_tr, train_seconds=train_s, **snaps)

    # ---- inference goldens ---------------------------------------------------
    gold = {}
    n_inf = 200
    t2 = time.time()
    gold["c3_counts_200"] = np.stack([run_presentation(x, w_fix, bank, cfg) for x in c3_img[:n_inf]])
    gold["c3_ms_per_img_1core"] = (time.time() - t2) * 1e3 / n_inf
    cfg75 = dataclasses.replace(cfg, t=0.075)
    gold["c4_counts_t75_100"] = np.stack([run_presentation(x, w_fix, bank, cfg75) for x in c4_img[:100]])
    cfg01 = dataclasses.replace(cfg, dt=1e-4)
    gold["c3_counts_dt01_12"] = np.stack([run_presentation(x, w_fix, bank, cfg01) for x in c3_img[:12]])
    # random weights: drives every output, exercises inhibition
    rng = np.random.default_rng(99)
    w_rand = rng.uniform(0, 1, size=(8112, 10)) * 5e-11 * (0.5 + np.arange(10) / 9.0)
    gold["w_rand"] = w_rand
    gold["c3_counts_wrand_40"] = np.stack([run_presentation(x, w_rand, bank, cfg) for x in c3_img[:40]])
    cfg_noinh = dataclasses.replace(cfg, inhibition_weight=0.0)
    gold["c3_counts_wrand_noinh_20"] = np.stack([run_presentation(x, w_rand, bank, cfg_noinh) for x in c3_img[:20]])

    # full rasters for a few images (hidden spike counts per neuron + output spikes)
    for k in range(4):
        rec = forward_pass(c3_img[k], w_fix, bank, cfg)
        gold[f"rec{k}_hidden_counts"] = np.array([len(s) for s in rec.hidden_spikes], dtype=np.int32)
        hm = np.zeros((cfg.n_steps, 8112), dtype=bool)
        for nidx, steps in enumerate(rec.hidden_spikes):
            hm[steps, nidx] = True
        gold[f"rec{k}_hidden_bits"] = np.packbits(hm, axis=1)
        om = np.zeros((cfg.n_steps, 10), dtype=bool)
        for l, steps in enumerate(rec.output_spikes):
            om[steps, l] = True
        gold[f"rec{k}_out"] = om
    # hidden currents (conv) for image 0: bit-exact target of the stencil
    gold["c3_0_hidden_currents"] = hidden_current_series(c3_img[0], bank, cfg)

    # input tables
    spk, ctab = _input_tables(cfg.encoding, cfg.input_lif, cfg.dt, cfg.n_steps)
    gold["table_dt1_spk"] = spk.copy()
    gold["table_dt1_c"] = ctab.copy()
    spk, ctab = _input_tables(cfg01.encoding, cfg01.input_lif, cfg01.dt, cfg01.n_steps)
    gold["table_dt01_sha"] = np.frombuffer(hashlib.sha256(ctab.tobytes()).digest(), dtype=np.uint8)
    gold["table_dt01_spkcount"] = spk.sum(axis=0)
    gold["table_dt01_c_rows"] = ctab[::97].copy()

    # training goldens: teacher-forced per-image steps from reference snapshots
    tf = {}
    for name in ("w_after_5", "w_after_100"):
        i = int(name.split("_")[-1])
        j = order[i]
        w_next, cts = train_presentation(c2_img[j], int(c2_lab[j]), snaps[name], bank, cfg, learn)
        tf[f"tf_{name}_dw"] = (w_next - snaps[name]) / learn.learning_rate
        tf[f"tf_{name}_counts"] = cts
    # dt = 0.1 ms training on 3 images from zero
    w01 = zero_weights()
    c01 = []
    for i in range(3):
        j = order[i]
        w01, cts = train_presentation(c2_img[j], int(c2_lab[j]), w01, bank, cfg01, learn)
        c01.append(cts)
    tf["train_dt01_w3"] = w01
    tf["train_dt01_counts3"] = np.stack(c01)
    gold.update(tf)

    np.savez_compressed(os.path.join(GOLD, "reference_golden.npz"), **gold)
    print(f"done in {time.time()-t0:.1f}s")
    for f in (os.path.join(DATA, "workloads.npz"), os.path.join(DATA, "w_fix.npz"),
              os.path.join(GOLD, "reference_golden.npz")):
        print(f, os.path.getsize(f) // 1024, "KiB")


if __name__ == "__main__":
    main()
