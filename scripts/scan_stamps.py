"""Per-step clock64 deltas of one image's output scan (image 40 of the c2
order) in the plain cluster kernel (mode 3) and the speculative one (mode 4);
needs a -DSNN_SCAN_STAMPS=40 build (scripts/build_variant.py)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
n = 100
order = d["c2_order"][:n]
imgs = torch.from_numpy(d["c2_images"][order].reshape(n, -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
f = eng.lib.snn_debug_scan_stamps
f.argtypes = [ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
res = {}
for mode in (3, 4):
    eng.lib.snn_set_normad_cluster(mode)
    for rep in range(3):
        dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        cnt, status = eng.train(c, imgs, labs, dw)
        torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 256)()
    f(buf, 256)
    st = np.array(buf[:101], dtype=np.int64)
    dd = np.diff(st)
    res[mode] = dd
    print(f"mode {mode}: total {st[100] - st[0]} cycles, per step mean {dd.mean():.0f} median {np.median(dd):.0f} "
          f"min {dd.min()} max {dd.max()}", flush=True)
eng.lib.snn_set_normad_cluster(4)
print("step  mode3  mode4")
for s in range(100):
    print(f"{s:4d} {res[3][s]:6d} {res[4][s]:6d}")
