"""Where the batch-1 run_presentation time goes (T = 75 ms): weights check,
image coercion, graph replay + copies."""
import dataclasses, os, sys, time, statistics
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import api  # noqa: E402
from paper_1711_03637_b200.engine import get_engine  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
cfg = dataclasses.replace(sd.NetworkConfig(), t=0.075)
bank = sd.default_filter_bank()
eng = get_engine()
imgs = d["c4_images"]
for im in imgs[:20]:
    sd.run_presentation(im, w, bank, cfg)
def med(f, k=300):
    ts = []
    for i in range(k):
        t0 = time.perf_counter(); f(i); ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6
print(f"run_presentation      {med(lambda i: sd.run_presentation(imgs[i % 500], w, bank, cfg)):8.1f} us")
print(f"eng.weights (compare) {med(lambda i: eng.weights(w, check=api._weights)):8.1f} us")
print(f"np.array_equal       {med(lambda i: np.array_equal(w, eng._w_host)):8.1f} us")
wb = w.tobytes()
print(f"bytes compare         {med(lambda i: w.tobytes() == wb):8.1f} us")
print(f"memoryview compare    {med(lambda i: memoryview(w).cast('B') == memoryview(eng._w_host).cast('B')):8.1f} us")
print(f"as_pixel_image        {med(lambda i: api.as_pixel_image(imgs[i % 500])):8.1f} us")
c = api._consts_cached(cfg, bank)
print(f"_consts_cached        {med(lambda i: api._consts_cached(cfg, bank)):8.1f} us")
print(f"infer_one             {med(lambda i: eng.infer_one(c, imgs[i % 500])):8.1f} us")
