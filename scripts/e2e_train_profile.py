import os, sys, time
import numpy as np
ROOT = "/root/repo"
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
order = d["c2_order"]
imgs, labs = d["c2_images"][order], d["c2_labels"][order]
cfg, bank, learn = sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig()
for rep in range(6):
    t0 = time.perf_counter()
    w, st = sd.train_epoch(imgs, labs, sd.zero_weights(), bank, cfg, learn)
    print(f"train_epoch e2e: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
import cProfile, pstats
cProfile.run("sd.train_epoch(imgs, labs, sd.zero_weights(), bank, cfg, learn)", "/tmp/prof.out")
pstats.Stats("/tmp/prof.out").sort_stats("cumtime").print_stats(15)
