"""k_output_dist vs k_output (snn_set_output_dist 1 / 0): counts, output
raster and traces of the 10,000 c3 images bit for bit, and the output-stage time."""
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
n = 10000
x = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
for e in evs:
    e.record(eng.stream)
arr = (ctypes.c_void_p * 7)(*[e.cuda_event for e in evs])
res = {}
for mode in (0, 1):
    eng.lib.snn_set_output_dist(mode)
    o = eng.infer(c, x, w, trace=True)
    eng.stream.synchronize()
    o2 = eng.infer(c, x, w, raster=True)
    eng.stream.synchronize()
    res[mode] = (o["counts"].cpu().numpy(), o["ff"].cpu().numpy(), o["v_out"].cpu().numpy(), o2["out_raster"].cpu().numpy())
    ts = []
    for rep in range(23):
        eng.lib.snn_profile_stage_events(arr, 6)
        eng.infer(c, x, w)
        eng.lib.snn_profile_stage_events(None, 0)
        evs[5].synchronize()
        if rep >= 3:
            ts.append(evs[4].elapsed_time(evs[5]))
    print(f"output_dist={mode}: k_output {statistics.median(ts):.4f} ms", flush=True)
eng.lib.snn_set_output_dist(1)
for k, name in enumerate(("counts", "ff", "v_out", "out_raster")):
    print(name, "equal:", bool(np.array_equal(res[0][k], res[1][k])))
