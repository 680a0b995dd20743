"""Throughput at the paper's dt = 0.1 ms (N = 1,000 steps): batched inference
(c3 images, W_fix) and NormAD training (c2 order, from zero weights)."""
import dataclasses, os, sys, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
cfg = dataclasses.replace(sd.NetworkConfig(), dt=1e-4)
bank = sd.default_filter_bank()
c = make_consts(cfg, bank, sd.LearnConfig())
w = torch.from_numpy(np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]).cuda()
for n in (10000,):
    x = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
    ts = []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream); eng.infer(c, x, w); e1.record(eng.stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"dt=0.1ms inference n={n}: {statistics.median(ts[2:]):.2f} ms  ({n / statistics.median(ts[2:]) * 1e3:.0f} img/s)")
order = d["c2_order"][:200]
imgs = torch.from_numpy(d["c2_images"][order].reshape(len(order), -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
for mode in (1, 0):
    eng.lib.snn_set_normad_cluster(mode)
    ts = []
    for rep in range(4):
        dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream); eng.train(c, imgs, labs, dw); e1.record(eng.stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"dt=0.1ms training cluster={mode}: {statistics.median(ts[1:]) / len(order) * 1e3:.1f} us/image "
          f"({len(order) / statistics.median(ts[1:]) * 1e3:.0f} img/s)")
eng.lib.snn_set_normad_cluster(4)
