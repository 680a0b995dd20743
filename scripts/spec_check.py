"""The speculative-scan NormAD kernel (snn_set_normad_cluster(4)) against the
plain cluster kernel (3): weights and per-image counts bit for bit over the
c2 epoch, the number of redone scans (d_status[3]) and the time per image."""
import os, statistics, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
order = np.resize(d["c2_order"], n)  # the 1,000-image c2 set, repeated past its end
imgs = torch.from_numpy(d["c2_images"][order].reshape(n, -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
res = {}
for mode in (3, 4):
    eng.lib.snn_set_normad_cluster(mode)
    ts = []
    for rep in range(6):
        dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        cnt, status = eng.train(c, imgs, labs, dw)
        e1.record(eng.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = status.cpu().numpy()
    res[mode] = (dw.cpu().numpy(), cnt.cpu().numpy())
    print(f"mode {mode}: {statistics.median(ts[2:]) * 1e3 / n:.2f} us/image  status {st}", flush=True)
eng.lib.snn_set_normad_cluster(4)
w3, w1 = res[3][0], res[4][0]
print("weights bitwise equal:", bool(np.array_equal(w3, w1)), " max|dw|", float(np.abs(w3 - w1).max()))
print("counts equal:", bool(np.array_equal(res[3][1], res[4][1])))
