"""One-warp timing of the serial output-layer scan (scripts/scan_micro.cu) on
realistic feed-forward inputs G (hidden rasters of c3 images under W_fix),
plus the FP64 dependent DADD+DMUL latency."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import _native  # noqa: E402
from paper_1711_03637_b200.engine import make_consts  # noqa: E402

so = os.path.join(ROOT, "scripts", "libscan_micro.so")
if not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                    "-o", so, os.path.join(ROOT, "scripts", "scan_micro.cu")], check=True)
lib = ctypes.CDLL(so)
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))
w = w[w.files[0]]
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
n_img = 16
Gs = []
for i in range(n_img):
    rec = sd.forward_pass(d["c3_images"][i], w, bank, cfg)
    m = np.zeros((cfg.n_steps, 8112))
    for k, ts in enumerate(rec.hidden_spikes):
        m[ts, k] = 1.0
    Gs.append(m @ w)
if os.environ.get("SCAN_W_TRAIN"):
    # weights after 40 online NormAD images from zero (the training regime)
    wt, _ = sd.train_epoch(d["c2_images"][d["c2_order"][:40]], d["c2_labels"][d["c2_order"][:40]],
                           sd.zero_weights(), bank, cfg, sd.LearnConfig())
    Gs = []
    for i in range(n_img):
        rec = sd.forward_pass(d["c2_images"][d["c2_order"][40 + i]], wt, bank, cfg)
        m = np.zeros((cfg.n_steps, 8112))
        for k, ts in enumerate(rec.hidden_spikes):
            m[ts, k] = 1.0
        Gs.append(m @ wt)
G = torch.from_numpy(np.stack(Gs)).cuda()
counts = torch.zeros((n_img, 10), dtype=torch.int32, device="cuda")
cyc = torch.zeros(4, dtype=torch.int64, device="cuda")
out = torch.zeros(32, dtype=torch.float64, device="cuda")
c = make_consts(cfg, bank)
iters = 4096
lib.micro_lat(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(cyc.data_ptr()), iters)
lib.micro_lat(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(cyc.data_ptr()), iters)
print(f"FP64 dependent DADD->DMUL pair: {cyc[0].item() / iters:.1f} cycles ({cyc[0].item() / iters / 2:.1f} per op)")
for mode, name in enumerate(("LDS.64 chase", "STS+syncwarp+LDS", "DSETP+VOTE+select (incl 1 DADD)", "SHFL f64", "DADD")):
    for _ in range(2):
        lib.micro_probe(mode, iters, ctypes.c_void_p(cyc.data_ptr()), ctypes.c_void_p(out.data_ptr()))
    print(f"probe {name}: {cyc[0].item() / iters:.1f} cycles/iter")
lib.micro_pingpong(iters, ctypes.c_void_p(cyc.data_ptr()))
lib.micro_pingpong(iters, ctypes.c_void_p(cyc.data_ptr()))
print(f"cross-warp ping-pong (shared memory flag): {cyc[0].item() / iters:.1f} cycles per round trip")
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
for _ in range(2):
    lib.micro_pingbar(iters, ctypes.c_void_p(cyc.data_ptr()), ctypes.c_void_p(sink.data_ptr()))
print(f"cross-warp ping-pong (named barriers): {cyc[0].item() / iters:.1f} cycles per round trip")
N = cfg.n_steps
VARIANTS = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "1"])]
res = {}
for variant in VARIANTS:
    om = torch.zeros((n_img, N), dtype=torch.int16, device="cuda")
    vv = torch.zeros((n_img, 10), dtype=torch.float64, device="cuda")
    for threads in (32,):
        for _ in range(2):
            lib.micro_scan(ctypes.byref(c), ctypes.c_void_p(G.data_ptr()), n_img, ctypes.c_void_p(counts.data_ptr()),
                           ctypes.c_void_p(cyc.data_ptr()), threads, variant, ctypes.c_void_p(om.data_ptr()),
                           ctypes.c_void_p(vv.data_ptr()))
        per_step = cyc[1].item() / (n_img * N)
        print(f"variant {variant} scan ({threads} threads/CTA): {per_step:.1f} cycles/step; output spikes/image "
              f"{counts.sum().item() / n_img:.1f}")
    res[variant] = (om.cpu().numpy().copy(), vv.cpu().numpy().copy(), counts.cpu().numpy().copy())
om0, v0, c0 = res[VARIANTS[0]]
for vv_ in VARIANTS[1:]:
    om1, v1, c1 = res[vv_]
    print(f"variant {vv_} vs {VARIANTS[0]}: masks identical:", np.array_equal(om0, om1), " v identical:",
          np.array_equal(v0.view(np.int64), v1.view(np.int64)), " counts identical:", np.array_equal(c0, c1))
pc = np.array([bin(int(x) & 0x3FF).count("1") for x in om0.ravel()])
print("steps with 0/1/2+ output spikes:", (pc == 0).sum(), (pc == 1).sum(), (pc >= 2).sum())
