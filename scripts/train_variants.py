"""Time the NormAD epoch (c2, 1,000 images) under the snn_set_normad_cluster modes."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
order = d["c2_order"]
imgs = torch.from_numpy(d["c2_images"][order].reshape(1000, -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
ref = None
for mode in (1, 2, 0, 1, 2):
    eng.lib.snn_set_normad_cluster(mode)
    ts = []
    for rep in range(3):
        dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream); eng.train(c, imgs, labs, dw); e1.record(eng.stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    w = dw.cpu().numpy()
    ref = w if ref is None else ref
    print(f"mode {mode}: {min(ts):.2f} ms  {1000 / min(ts) * 1e3:.0f} img/s  max|dW vs mode1| {np.abs(w - ref).max():.3e}", flush=True)
eng.lib.snn_set_normad_cluster(4)
