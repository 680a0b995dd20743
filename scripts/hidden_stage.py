"""Median device time of the guard-band hidden layer and of its float64 redo
(library stage events 2 -> 6 -> 3) over 20 calls of an n-image c3 batch (argv[1], default 10,000)."""
import ctypes, os, statistics, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank())
w = torch.from_numpy(np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]).cuda()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
x = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
for e in evs:
    e.record(eng.stream)
arr = (ctypes.c_void_p * 7)(*[e.cuda_event for e in evs])
gb, fix = [], []
for rep in range(23):
    eng.lib.snn_profile_stage_events(arr, 7)
    eng.infer(c, x, w)
    eng.lib.snn_profile_stage_events(None, 0)
    evs[5].synchronize()
    if rep >= 3:
        gb.append(evs[2].elapsed_time(evs[6]))
        fix.append(evs[6].elapsed_time(evs[3]))
print(f"k_hidden_gb {statistics.median(gb):.4f} ms  k_hidden_fix {statistics.median(fix):.4f} ms")
