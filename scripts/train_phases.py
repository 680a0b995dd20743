"""Per-phase cycle breakdown of the cluster NormAD kernel (leader CTA clock64 stamps)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_03637_b200 import build as _build  # noqa: E402
os.environ["SNN_B200_LIB"] = _build.build_profile()  # hooks are compiled only into the profile build
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
names = ["G partials", "B1", "gather G", "scan", "sigma", "R adjoint", "B2", "copy R", "dW", "B3", "commit", "next"]
d_ = np.diff(k[:, :12], axis=1)
nxt = k[1:, 0] - k[:-1, 11]
print("cycles per phase (median over images 4..63):")
for i, n in enumerate(names[:11]):
    print(f"  {n:12s} {np.median(d_[:, i]):8.0f}")
print(f"  {'to next img':12s} {np.median(nxt):8.0f}")
print("scan cycles per image:", d_[:, 3].tolist()[:8])
print("scan warp loop (median):", np.median(k[:, 12] - k[:, 3]), " stage warps (median):", np.median(k[:, 13] - k[:, 3]))
tot = np.median(k[1:, 0] - k[:-1, 0])
print(f"  per image    {tot:8.0f} cycles = {tot / 1.965e3:.2f} us at 1965 MHz")
