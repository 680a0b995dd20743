"""60,000-image batch (6 x config 3, crosses the 4 GB workspace chunking): counts equal the reference's; steady-state e2e throughput."""
import os, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1711_03637_b200 as sd
d = np.load("/root/repo/data/workloads.npz"); w = np.load("/root/repo/data/w_fix.npz")["w_fix"]
ref = np.load("/root/repo/tests/golden/c3_counts_reference.npz")["counts"].astype(np.int64)
imgs = np.concatenate([d["c3_images"]] * 6)
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
sd.batch_counts(imgs[:1000], w, bank, cfg)
for rep in range(3):  # the first call at this size allocates the workspace and pinned staging
    t0 = time.perf_counter(); got = sd.batch_counts(imgs, w, bank, cfg); t = time.perf_counter() - t0
print("60k images:", got.shape, "equal to 6x reference:", np.array_equal(got, np.concatenate([ref] * 6)), f"{t*1e3:.1f} ms, {len(imgs)/t/1e6:.2f} M img/s e2e")
