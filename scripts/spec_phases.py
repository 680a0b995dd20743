"""Phase clocks of the speculative NormAD kernel (profiling variant built with
-DSNN_SPEC_PROFILE; SNN_B200_LIB points at it)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
eng.lib.snn_set_normad_cluster(4)  # the speculative kernel
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
k = clk.cpu().numpy()[4:60].astype(np.float64)
names = {1: "scan warp done", 2: "R + stage", 3: "dW", 4: "partials", 5: "barrier A", 6: "gathers",
         7: "E bound", 8: "(1)", 12: "check loop", 13: "check barrier", 9: "check (2)", 10: "handover"}
print("cycles since loop top (median over images 4..59):")
for j, nm in names.items():
    print(f"  {nm:16s} {np.median(k[:, j] - k[:, 0]):8.0f}")
print("  per image       ", np.median(k[1:, 0] - k[:-1, 0]))
print("raw (images 10..13, relative to each loop top):")
for i in range(6, 10):
    print("  ", [int(x) for x in (k[i, :16] - k[i, 0])])
