"""Cost of each phase of the cluster NormAD kernel by ablation (snn_normad_skip;
results are wrong while a phase is skipped -- timing only).  Runs the profiling
build (build.py --profile), whose serial scan compiles differently from the
product kernel: absolute times are higher than bench.py's, differences indicative."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_03637_b200 import build as _build  # noqa: E402
os.environ["SNN_B200_LIB"] = _build.build_profile()  # hooks are compiled only into the profile build
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200.engine import get_engine, make_consts  # noqa: E402
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
eng = get_engine()
c = make_consts(sd.NetworkConfig(), sd.default_filter_bank(), sd.LearnConfig())
order = d["c2_order"]
imgs = torch.from_numpy(d["c2_images"][order].reshape(1000, -1).copy()).cuda()
labs = torch.from_numpy(d["c2_labels"][order].astype(np.uint8)).cuda()
def run(mask):
    eng.lib.snn_normad_skip(mask)
    ts = []
    for rep in range(3):
        dw = torch.zeros((8112, 10), dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream); eng.train(c, imgs, labs, dw); e1.record(eng.stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    eng.lib.snn_normad_skip(0)
    return min(ts) / 1000 * 1e3  # us per image
base = run(0)
print(f"full: {base:.2f} us/image")
for mask, name in ((1, "output scan"), (2, "R adjoint"), (4, "dW"), (8, "G partials"), (16, "G gather"), (31, "all five")):
    t = run(mask)
    print(f"  without {name:12s}: {t:6.2f} us/image  (phase ~{base - t:5.2f} us)", flush=True)
