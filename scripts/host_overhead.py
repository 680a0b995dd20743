"""Host-side cost of one batch_counts call on the 10,000 c3 images, split:
device time of the call (events) vs wall time of each Python step."""
import os, sys, time, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import api  # noqa: E402
from paper_1711_03637_b200.engine import get_engine  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
imgs = np.ascontiguousarray(d["c3_images"].reshape(10000, -1))
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
eng = get_engine()
for _ in range(3):
    sd.batch_counts(imgs, w, bank, cfg)
T = {k: [] for k in ("validate", "consts", "weights", "upload", "infer_launch", "wait_device", "fetch", "total")}
for rep in range(15):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = api.as_pixel_batch(imgs); t1 = time.perf_counter()
    c = api._consts_cached(cfg, bank); t2 = time.perf_counter()
    with eng.lock:
        d_w = eng.weights(w, check=api._weights); t3 = time.perf_counter()
        d_img = eng.upload("images", x).view(len(x), -1); t4 = time.perf_counter()
        counts = eng.infer(c, d_img, d_w)["counts"]; t5 = time.perf_counter()
        eng.stream.synchronize(); t6 = time.perf_counter()
        out = api._fetch(eng, counts); t7 = time.perf_counter()
    for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6, t7 - t0)):
        T[k].append(v * 1e3)
print("  ".join(f"{k} {statistics.median(v):.3f}" for k, v in T.items()), "ms")
