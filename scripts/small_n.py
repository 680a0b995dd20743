"""Hidden-layer time of the guard-band (mode 1) and the float64 (mode 3)
kernels for small batches -- picks the batch size below which the float64
kernel is faster (its setup is lighter and it needs no redo launch)."""
import subprocess, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import ctypes, statistics
import numpy as np
import torch
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank())
w = torch.from_numpy(np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]).cuda()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
for e in evs:
    e.record(eng.stream)
arr = (ctypes.c_void_p * 7)(*[e.cuda_event for e in evs])
for n in (1, 4, 16, 64, 148, 300, 600, 1250):
    x = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
    res = []
    for mode in (1, 3):
        eng.lib.snn_set_hidden_resident(mode)
        hs, cs = [], []
        for rep in range(25):
            eng.lib.snn_profile_stage_events(arr, 6)
            eng.infer(c, x, w)
            eng.lib.snn_profile_stage_events(None, 0)
            evs[5].synchronize()
            if rep >= 5:
                hs.append(evs[2].elapsed_time(evs[3])); cs.append(evs[0].elapsed_time(evs[5]))
        res.append((statistics.median(hs), statistics.median(cs)))
    eng.lib.snn_set_hidden_resident(1)
    print(f"n={n:5d}  guard band: hidden {res[0][0]*1e3:7.1f} us call {res[0][1]*1e3:7.1f} us   "
          f"float64: hidden {res[1][0]*1e3:7.1f} us call {res[1][1]*1e3:7.1f} us", flush=True)
