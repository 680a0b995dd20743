"""Per-kernel device times of the 10,000-image c3 call (library stage events,
median of 20) -- for A/B of builds (scripts/variants.sh)."""
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
names = ["prep", "scan", "hidden", "gsum", "output"]
per = {k: [] for k in names + ["call"]}
for rep in range(23):
    eng.lib.snn_profile_stage_events(arr, 6)
    eng.infer(c, x, w)
    eng.lib.snn_profile_stage_events(None, 0)
    evs[5].synchronize()
    if rep >= 3:
        for k, nm in enumerate(names):
            per[nm].append(evs[k].elapsed_time(evs[k + 1]))
        per["call"].append(evs[0].elapsed_time(evs[5]))
print(f"n={n} " + "  ".join(f"{k} {statistics.median(v):.4f}" for k, v in per.items()) + " ms", flush=True)
