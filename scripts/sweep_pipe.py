"""Sweep snn_set_hidden_resident x snn_set_pipeline(images_per_subbatch, hidden_ctas_per_sm) on the c3
workload (10k images)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402

d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
gold = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))["c3_counts_200"]
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank())
imgs = torch.from_numpy(d["c3_images"].reshape(10000, -1).copy()).cuda()
dw = torch.from_numpy(w.copy()).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for res, per, ctas in [(1, 0, 0), (1, 2048, 0), (1, 3334, 0), (0, 0, 0), (0, 1024, 3), (0, 2048, 3), (0, 1024, 4), (0, 2048, 4), (0, 3334, 4), (0, 2048, 2)]:
    eng.lib.snn_set_hidden_resident(res)
    eng.lib.snn_set_pipeline(per, ctas)
    for _ in range(3):
        out = eng.infer(c, imgs, dw)["counts"]
    ts = []
    for _ in range(10):
        with torch.cuda.stream(eng.stream):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        out = eng.infer(c, imgs, dw)["counts"]
        e1.record(eng.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    o = out.cpu().numpy()
    ref = o if ref is None else ref
    print(f"res={res} per={per:5d} ctas={ctas}: {np.median(ts):.3f} ms  ({10000 / np.median(ts) * 1e3 / 1e6:.3f} M img/s)  "
          f"same={np.array_equal(o, ref)} gold200={np.array_equal(o[:200], gold)}", flush=True)
