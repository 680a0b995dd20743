"""Where the host-API batch inference time goes (10,000 c3 images)."""
import os, sys, time, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import api  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
imgs = d["c3_images"].reshape(10000, -1).copy()
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
eng = get_engine()
c = make_consts(cfg, bank)
def med(f, k=15):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts[3:]) * 1e3
d_img = api._to_device(eng, imgs); d_w = api._to_device(eng, w)
print(f"batch_counts (API)       {med(lambda: sd.batch_counts(imgs, w, bank, cfg)):.3f} ms")
print(f"_weights check           {med(lambda: api._weights(w)):.3f} ms")
print(f"_to_device images        {med(lambda: api._to_device(eng, imgs)):.3f} ms")
print(f"_to_device weights       {med(lambda: api._to_device(eng, w)):.3f} ms")
print(f"pin_memory images only   {med(lambda: torch.from_numpy(imgs).pin_memory()):.3f} ms")
pinned = torch.from_numpy(imgs).pin_memory()
print(f"H2D from pinned          {med(lambda: d_img.copy_(pinned, non_blocking=True)):.3f} ms")
print(f"H2D from pageable        {med(lambda: d_img.copy_(torch.from_numpy(imgs), non_blocking=False)):.3f} ms")
print(f"infer (device)           {med(lambda: eng.infer(c, d_img, d_w)):.3f} ms")
out = eng.infer(c, d_img, d_w)["counts"]
print(f"fetch counts             {med(lambda: api._fetch(eng, out)):.3f} ms")
