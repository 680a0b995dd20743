"""Device time of one snn_train call over the c2 epoch (1,000 images, the
bench's training workload) and over 3,000 images (the set repeated): median
of 5 calls, microseconds per image."""
import os, statistics, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
for n in (1000, 3000):
    order = np.resize(d["c2_order"], n)
    imgs = torch.from_numpy(d["c2_images"][order].reshape(n, -1).copy()).cuda()
    labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
    ts = []
    for rep in range(7):
        w = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        eng.train(c, imgs, labs, w)
        e1.record(eng.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={n}: {statistics.median(ts[2:]):.3f} ms, {statistics.median(ts[2:]) * 1e3 / n:.2f} us/image", flush=True)
