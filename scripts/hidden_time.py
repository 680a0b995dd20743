"""k_hidden alone (library events around its launch, un-pipelined call) on the
10,000-image c3 batch, median of 30 -- for A/B of builds (scripts/variants.sh)."""
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
x = torch.from_numpy(d["c3_images"].reshape(10000, -1).copy()).cuda()
lib = eng.lib
lib.snn_set_pipeline(0, 0)
eb, ea = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
eb.record(eng.stream); ea.record(eng.stream)
hk, call = [], []
for rep in range(33):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    lib.snn_profile_events(ctypes.c_void_p(eb.cuda_event), ctypes.c_void_p(ea.cuda_event))
    eng.infer(c, x, w)
    lib.snn_profile_events(None, None)
    e1.record(eng.stream); e1.synchronize()
    if rep >= 3:
        hk.append(eb.elapsed_time(ea)); call.append(e0.elapsed_time(e1))
print(f"k_hidden {statistics.median(hk):.4f} ms (min {min(hk):.4f})  call {statistics.median(call):.4f} ms")
