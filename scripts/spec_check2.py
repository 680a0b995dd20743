"""Training modes 1 (cluster, default), 3 and 4 (speculative scan) on the
same images: weights and per-image counts compared pairwise (first differing
image)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd
from paper_1711_03637_b200.engine import get_engine, make_consts
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
n = int(sys.argv[1])
order = np.resize(d["c2_order"], n)  # the 1,000-image c2 set, repeated past its end
imgs = torch.from_numpy(d["c2_images"][order].reshape(n, -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
res = {}
for mode in (1, 3, 4):
    eng.lib.snn_set_normad_cluster(mode)
    dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
    cnt, status = eng.train(c, imgs, labs, dw)
    torch.cuda.synchronize()
    res[mode] = (dw.cpu().numpy(), cnt.cpu().numpy(), status.cpu().numpy())
    print(mode, res[mode][2], flush=True)
eng.lib.snn_set_normad_cluster(4)
for a, b in ((1, 3), (1, 4), (3, 4)):
    ca, cb = res[a][1], res[b][1]
    diff = np.nonzero((ca != cb).any(axis=1))[0]
    print(f"{a} vs {b}: W equal {np.array_equal(res[a][0], res[b][0])}, first differing image {diff[:5]}, n diff {len(diff)}")
    if len(diff):
        i = diff[0]; print("   counts", ca[i], cb[i])
