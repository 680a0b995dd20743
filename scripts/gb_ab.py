"""A/B of the hidden-layer kernels on the 10,000-image c3 batch: k_hidden time
(library events around the hidden launches, un-pipelined call, median of 20),
the guard-band redo count, and the compact raster against the float64
kernel (snn_set_hidden_resident: 1 = guard band v2, 4 = guard band v1,
3 = float64 table-resident)."""
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
x = torch.from_numpy(d["c3_images"].reshape(n, -1).copy()).cuda()
lib = eng.lib
lib.snn_set_pipeline(0, 0)
modes = [int(a) for a in sys.argv[1:]] or [3, 4, 1]
ref = None
for mode in modes:
    lib.snn_set_hidden_resident(mode)
    o = eng.infer(c, x, w, raster=True)
    eng.stream.synchronize()
    nb = int(o["tile_base"][n].item()) * (-(-c.n_steps // 8)) * 512
    ras, cnt, redo = o["raster"][:nb].clone(), o["counts"].clone(), int(o["hidden_redo"].item())
    if ref is None:
        ref = (ras, cnt)
    same = bool(torch.equal(ras, ref[0])) and bool(torch.equal(cnt, ref[1]))
    eb, ea = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eb.record(eng.stream); ea.record(eng.stream)
    hk, call = [], []
    for rep in range(23):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        lib.snn_profile_events(ctypes.c_void_p(eb.cuda_event), ctypes.c_void_p(ea.cuda_event))
        eng.infer(c, x, w)
        lib.snn_profile_events(None, None)
        e1.record(eng.stream); e1.synchronize()
        if rep >= 3:
            hk.append(eb.elapsed_time(ea)); call.append(e0.elapsed_time(e1))
    print(f"mode {mode}: k_hidden {statistics.median(hk):.4f} ms (min {min(hk):.4f})  call "
          f"{statistics.median(call):.4f} ms  redo {redo}  raster+counts == mode {modes[0]}: {same}", flush=True)
lib.snn_set_hidden_resident(1)
