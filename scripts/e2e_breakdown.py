"""Where the host-API batch inference time goes (10,000 c3 images), and the
candidate ways to move the 7.8 MB of images to the device."""
import os, sys, time, statistics
from concurrent.futures import ThreadPoolExecutor
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import api  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
imgs = np.ascontiguousarray(d["c3_images"][:n].reshape(n, -1))
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
eng = get_engine()
c = make_consts(cfg, bank)
def med(f, k=15):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts[3:]) * 1e3
d_img = api._to_device(eng, imgs); d_w = api._to_device(eng, w)
pinned = torch.empty(imgs.nbytes, dtype=torch.uint8).pin_memory()
pn = pinned.numpy()
pool = ThreadPoolExecutor(4)
def threaded_copy():
    flat = imgs.reshape(-1)
    cuts = np.linspace(0, flat.size, 5).astype(int)
    list(pool.map(lambda k: np.copyto(pn[cuts[k]:cuts[k + 1]], flat[cuts[k]:cuts[k + 1]]), range(4)))
print(f"n={n}")
print(f"batch_counts (API)       {med(lambda: sd.batch_counts(imgs, w, bank, cfg)):.3f} ms")
print(f"as_pixel_batch           {med(lambda: api.as_pixel_batch(imgs)):.3f} ms")
print(f"_weights check           {med(lambda: api._weights(w)):.3f} ms")
print(f"eng.weights (cached)     {med(lambda: eng.weights(w, check=api._weights)):.3f} ms")
print(f"_to_device images        {med(lambda: api._to_device(eng, imgs)):.3f} ms")
print(f"pin_memory images only   {med(lambda: torch.from_numpy(imgs).pin_memory()):.3f} ms")
print(f"copyto persistent pinned {med(lambda: np.copyto(pn, imgs.reshape(-1))):.3f} ms")
print(f"4-thread copy to pinned  {med(threaded_copy):.3f} ms")
print(f"H2D from pinned          {med(lambda: d_img.view(-1).copy_(pinned, non_blocking=True)):.3f} ms")
print(f"H2D from pageable        {med(lambda: d_img.copy_(torch.from_numpy(imgs), non_blocking=False)):.3f} ms")
print(f"infer (device)           {med(lambda: eng.infer(c, d_img, d_w)):.3f} ms")
out = eng.infer(c, d_img, d_w)["counts"]
print(f"fetch counts             {med(lambda: api._fetch(eng, out)):.3f} ms")
print(f"make_consts              {med(lambda: make_consts(cfg, bank)):.3f} ms")
# pinning the caller's buffer in place
cr = torch.cuda.cudart()
def reg():
    cr.cudaHostRegister(imgs.ctypes.data, imgs.nbytes, 0)
    cr.cudaHostUnregister(imgs.ctypes.data)
print(f"cudaHostRegister+unreg   {med(reg):.3f} ms")
half = n // 2
def two_chunk():
    a = api.batch_counts(imgs[:half], w, bank, cfg)
    b = api.batch_counts(imgs[half:], w, bank, cfg)
print(f"2 sequential half calls  {med(two_chunk):.3f} ms")
