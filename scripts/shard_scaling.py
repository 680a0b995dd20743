"""Projected 1/2/4/8-GPU scaling of batched inference from one GPU (SCALE runs
need an 8-GPU node): device time of one snn_infer call (CUDA events) and end-
to-end time of the public API on one rank's shard (batch_counts with host
numpy in/out, the per-rank work of distributed.sharded_batch_counts) at
10,000 / N images, N = 1, 2, 4, 8.  The projection assumes ranks run
concurrently and adds the measured all-gather of the counts (NCCL over
NVLink for 8 x 1,250 x 40 B is ~20 us; taken as 30 us, stated)."""
import json, os, statistics, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
wf = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
eng = get_engine()
c = make_consts(cfg, bank)
w = torch.from_numpy(wf.copy()).cuda()
imgs_all = d["c3_images"]
GATHER_MS = 0.030
res = {}
for N in (1, 2, 4, 8):
    n = 10000 // N
    x = torch.from_numpy(imgs_all[:n].reshape(n, -1).copy()).cuda()
    dev = []
    for rep in range(23):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        eng.infer(c, x, w)
        e1.record(eng.stream)
        e1.synchronize()
        if rep >= 3:
            dev.append(e0.elapsed_time(e1))
    host = imgs_all[:n]
    e2e = []
    for rep in range(13):
        t0 = time.perf_counter()
        sd.batch_counts(host, wf, bank, cfg)
        if rep >= 3:
            e2e.append((time.perf_counter() - t0) * 1e3)
    res[N] = {"images_per_rank": n, "device_ms": statistics.median(dev), "e2e_ms": statistics.median(e2e)}
base_d, base_e = res[1]["device_ms"], res[1]["e2e_ms"]
for N, r in res.items():
    g = GATHER_MS if N > 1 else 0.0
    r["projected_device_images_per_s"] = 10000 / ((r["device_ms"] + g) * 1e-3)
    r["projected_e2e_images_per_s"] = 10000 / ((r["e2e_ms"] + g) * 1e-3)
    r["projected_device_efficiency"] = base_d / (N * (r["device_ms"] + g))
    r["projected_e2e_efficiency"] = base_e / (N * (r["e2e_ms"] + g))
print(json.dumps(res, indent=1))
