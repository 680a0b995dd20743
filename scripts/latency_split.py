"""Batch-1 inference (T = 75 ms) split: k_hidden (library events) vs the rest of the call."""
import dataclasses, sys, statistics, ctypes
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1711_03637_b200 as sd
from paper_1711_03637_b200.engine import get_engine, make_consts
d = np.load("/root/repo/data/workloads.npz"); w = torch.from_numpy(np.load("/root/repo/data/w_fix.npz")["w_fix"]).cuda()
cfg = dataclasses.replace(sd.NetworkConfig(), t=0.075); bank = sd.default_filter_bank()
eng = get_engine(); c = make_consts(cfg, bank)
x = torch.from_numpy(d["c4_images"][:1].reshape(1, -1).copy()).cuda()
hb, ha = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
hb.record(eng.stream); ha.record(eng.stream); torch.cuda.synchronize()  # create the events
eng.lib.snn_profile_events(ctypes.c_void_p(hb.cuda_event), ctypes.c_void_p(ha.cuda_event))
tot, hid = [], []
for i in range(200):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream); eng.infer(c, x, w); e1.record(eng.stream); e1.synchronize()
    tot.append(e0.elapsed_time(e1) * 1e3); hid.append(hb.elapsed_time(ha) * 1e3)
eng.lib.snn_profile_events(None, None)
print(f"batch-1 infer (events): total p50 {statistics.median(tot):.1f} us; k_hidden {statistics.median(hid):.1f} us; "
      f"rest (prep, scan, gsum, output + gaps) {statistics.median(tot) - statistics.median(hid):.1f} us")
