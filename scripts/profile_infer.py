"""Minimal inference driver for ncu captures: 2 warm-up passes + 1 profiled pass."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
train = "--train" in sys.argv
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
eng = get_engine()
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
if train:
    c = make_consts(cfg, bank, sd.LearnConfig())
    order = d["c2_order"][:n]
    imgs = torch.from_numpy(d["c2_images"][order].reshape(len(order), -1).copy()).cuda()
    labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
    for _ in range(3):
        dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        eng.train(c, imgs, labs, dw)
else:
    c = make_consts(cfg, bank)
    imgs = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
    dw = torch.from_numpy(w.copy()).cuda()
    for _ in range(3):
        eng.infer(c, imgs, dw)
torch.cuda.synchronize()
print("done")
