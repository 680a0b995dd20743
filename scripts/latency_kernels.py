"""A few batch-1 run_presentation calls (T = 75 ms) for an ncu launch list."""
import dataclasses, sys
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1711_03637_b200 as sd
d = np.load("data/workloads.npz"); w = np.load("data/w_fix.npz")["w_fix"]
cfg = dataclasses.replace(sd.NetworkConfig(), t=0.075); bank = sd.default_filter_bank()
for x in d["c4_images"][:6]:
    sd.run_presentation(x, w, bank, cfg)
