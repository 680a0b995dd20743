"""Per-neuron hidden spike counts of 1,000 config-3 images (every 10th of the
10,000 images of synthetic_dataset(1000, seed=2000), T = 100 ms, dt = 1 ms,
weights W_fix), generated FROM THE REFERENCE's own forward_pass
(network.py:329-346: SpikeRecord.hidden_spikes, one list of step indices per
hidden neuron), with its output counts:

    python oracle/gen_hidden_counts.py  ->  tests/golden/c3_hidden_counts_reference.npz

hidden_counts[i, k] = len(record.hidden_spikes[k]) of image idx[i] (uint8;
a neuron fires at most every 4th step, so at most 25 times);
first_spike[i, k] = its first spike step (-1 if none), a second per-neuron
check that is independent of the count.  Test infrastructure only.
"""
from __future__ import annotations

import os
import sys
import time
from multiprocessing import Pool

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "c3_hidden_counts_reference.npz")
STRIDE = 10


def _one(args):
    img, w = args
    from spikedigits.filters import default_filter_bank
    from spikedigits.network import NetworkConfig, forward_pass
    rec = forward_pass(img, w, default_filter_bank(), NetworkConfig())
    cnt = np.array([len(s) for s in rec.hidden_spikes], dtype=np.uint8)
    first = np.array([s[0] if len(s) else -1 for s in rec.hidden_spikes], dtype=np.int8)
    return cnt, first, np.asarray(rec.output_counts, dtype=np.int16)


def main():
    sys.path.insert(0, REF)
    d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
    w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
    idx = np.arange(0, len(d["c3_images"]), STRIDE)
    t0 = time.time()
    with Pool(os.cpu_count() or 8, initializer=sys.path.insert, initargs=(0, REF)) as pool:
        res = pool.map(_one, [(d["c3_images"][i], w) for i in idx], chunksize=8)
    cnt = np.stack([r[0] for r in res])
    first = np.stack([r[1] for r in res])
    out = np.stack([r[2] for r in res])
    np.savez_compressed(OUT, idx=idx.astype(np.int32), hidden_counts=cnt, first_spike=first, output_counts=out)
    print(cnt.shape, int(cnt.sum()), f"{time.time() - t0:.0f} s ->", OUT)


if __name__ == "__main__":
    main()
