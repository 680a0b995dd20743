"""Device time of the batch-1 serving graph (T = 75 ms): per replay with events, and back to back."""
import dataclasses, os, sys, time, statistics
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1711_03637_b200 as sd
from paper_1711_03637_b200 import api
from paper_1711_03637_b200.engine import get_engine
d = np.load("/root/repo/data/workloads.npz"); w = np.load("/root/repo/data/w_fix.npz")["w_fix"]
cfg = dataclasses.replace(sd.NetworkConfig(), t=0.075); bank = sd.default_filter_bank()
eng = get_engine(); imgs = d["c4_images"]
for x in imgs[:50]: sd.run_presentation(x, w, bank, cfg)
c = api._consts_cached(cfg, bank)
gr = eng._graphs[bytes(c)]
ts = []
for i in range(300):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gr["img_np"][:] = imgs[i % 500].reshape(-1)
    with torch.cuda.stream(eng.stream):
        e0.record(eng.stream); gr["g"].replay(); e1.record(eng.stream)
    e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
print(f"graph replay (device, events): p50 {statistics.median(ts):.1f} us, min {min(ts):.1f} us")
# back-to-back replays without sync in between (device throughput of the batch-1 chain)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(eng.stream):
    e0.record(eng.stream)
    for i in range(200): gr["g"].replay()
    e1.record(eng.stream)
e1.synchronize(); print(f"200 back-to-back replays: {e0.elapsed_time(e1)*1e3/200:.1f} us each")
