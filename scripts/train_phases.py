"""Per-phase cycle breakdown of the cluster NormAD kernel (leader CTA clock64 stamps)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_03637_b200 import build as _build  # noqa: E402
if not os.environ.get("SNN_B200_LIB"):  # hooks are compiled only into the profile build
    os.environ["SNN_B200_LIB"] = _build.build_profile()
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402

d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
order = d["c2_order"][:200]
imgs = torch.from_numpy(d["c2_images"][order].reshape(len(order), -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
clk = torch.zeros((64, 16), dtype=torch.int64, device="cuda")
for rep in range(3):
    dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
    eng.lib.snn_normad_phase_clocks(ctypes.c_void_p(clk.data_ptr() if rep == 2 else 0))
    eng.train(c, imgs, labs, dw)
    torch.cuda.synchronize()
eng.lib.snn_normad_phase_clocks(None)
k = clk.cpu().numpy()[4:64]
# stamps of k_normad_cl (normad_cl.cuh): 0 start, 1 partials done, 2 after B1,
# 3 G gathered, 12 scan warp done, 13 stage warps done, 4 scan section done,
# 5 after OMASK broadcast + B2, 6 sigma, 7 R adjoint, 9 dW committed
edges = [("G partials", 0, 1), ("B1", 1, 2), ("gather G", 2, 3), ("scan (warp 0)", 3, 12),
         ("scan section", 3, 4), ("bcast + B2", 4, 5), ("sigma", 5, 6), ("R adjoint", 6, 7), ("dW", 7, 9)]
print("cycles per phase (median over images 4..63):")
for name, a, b in edges:
    print(f"  {name:14s} {np.median(k[:, b] - k[:, a]):8.0f}")
nxt = k[1:, 0] - k[:-1, 9]
print(f"  {'to next img':14s} {np.median(nxt):8.0f}")
print("stage warps (median):", np.median(k[:, 13] - k[:, 3]))
tot = np.median(k[1:, 0] - k[:-1, 0])
print(f"  per image      {tot:8.0f} cycles = {tot / 1.965e3:.2f} us at 1965 MHz")
