"""Median wall time of eng.train over the c2 workload (1,000 images), after
warm-up; also the inference batch (10,000 images) -- for A/B of builds."""
import os, sys, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
c = make_consts(cfg, bank, sd.LearnConfig())
order = d["c2_order"]
imgs = torch.from_numpy(d["c2_images"][order].reshape(1000, -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
if os.environ.get("SNN_CLUSTER_MODE"):
    eng.lib.snn_set_normad_cluster(int(os.environ["SNN_CLUSTER_MODE"]))
ts = []
for rep in range(8):
    dw.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream); eng.train(c, imgs, labs, dw); e1.record(eng.stream); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"train: median {statistics.median(ts[3:]) * 1e3 / 1000:.2f} us/image  all {[round(t, 2) for t in ts]}")
w = torch.from_numpy(np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]).cuda()
x = torch.from_numpy(d["c3_images"].reshape(10000, -1).copy()).cuda()
ts = []
for rep in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream); eng.infer(c, x, w); e1.record(eng.stream); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"infer: median {statistics.median(ts[3:]):.3f} ms / 10k images")
