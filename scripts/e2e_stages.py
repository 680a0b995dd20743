"""Wall-clock stages of one host-API batch_counts call (10,000 c3 images):
where the time between the device call and the end-to-end number goes."""
import os, statistics, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import api  # noqa: E402
from paper_1711_03637_b200.engine import get_engine  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
imgs = np.ascontiguousarray(d["c3_images"][:10000].reshape(10000, -1))
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
eng = get_engine()
names = ["as_pixel_batch", "consts", "weights", "upload", "infer (enqueue)", "sync", "fetch (D2H + int64)"]
acc = {k: [] for k in names + ["total"]}
for rep in range(25):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    x = api.as_pixel_batch(imgs); t.append(time.perf_counter())
    c = api._consts_cached(cfg, bank); t.append(time.perf_counter())
    with eng.lock:
        d_w = eng.weights(w, check=api._weights); t.append(time.perf_counter())
        d_img = eng.upload("images", x).view(len(x), -1); t.append(time.perf_counter())
        out = eng.infer(c, d_img, d_w)["counts"]; t.append(time.perf_counter())
        eng.stream.synchronize(); t.append(time.perf_counter())
        r = api._fetch(eng, out, np.int64); t.append(time.perf_counter())
    if rep >= 5:
        for k, nm in enumerate(names):
            acc[nm].append((t[k + 1] - t[k]) * 1e3)
        acc["total"].append((t[-1] - t[0]) * 1e3)
for k, v in acc.items():
    print(f"{k:16s} {statistics.median(v):.3f} ms")
