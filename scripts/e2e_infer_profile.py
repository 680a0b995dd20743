"""cProfile of the host-API batch inference call (distributed.sharded_batch_counts, 10,000 c3 images): where the host time goes around the device work."""
import os, sys, time, statistics, cProfile, pstats
import numpy as np, torch
ROOT = "/root/repo"; sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd
from paper_1711_03637_b200 import distributed as sdist
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
imgs = d["c3_images"]
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
for _ in range(5): sdist.sharded_batch_counts(imgs, w, bank, cfg)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); sdist.sharded_batch_counts(imgs, w, bank, cfg); ts.append(time.perf_counter() - t0)
print("api median ms", statistics.median(ts) * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): sdist.sharded_batch_counts(imgs, w, bank, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
