"""Output-layer device time (stage events 4 -> 5) with the lane-distributed
kernel (snn_set_output_dist(1)) and the replicated one (0) at several batch
sizes: where the crossover lies."""
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
evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
for e in evs:
    e.record(eng.stream)
arr = (ctypes.c_void_p * 7)(*[e.cuda_event for e in evs])
for n in (256, 625, 1250, 2500, 5000, 10000):
    x = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
    row = [f"n={n:5d}"]
    for mode in (1, 0):
        eng.lib.snn_set_output_dist(mode)
        t = []
        for rep in range(15):
            eng.lib.snn_profile_stage_events(arr, 6)
            eng.infer(c, x, w)
            eng.lib.snn_profile_stage_events(None, 0)
            evs[5].synchronize()
            if rep >= 3:
                t.append(evs[4].elapsed_time(evs[5]))
        row.append(f"{'dist' if mode else 'repl'} {statistics.median(t) * 1e3:.1f} us")
    eng.lib.snn_set_output_dist(1)
    print("  ".join(row), flush=True)
