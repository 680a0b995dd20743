import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1711_03637_b200 as sd
from paper_1711_03637_b200.engine import get_engine, make_consts
from paper_1711_03637_b200.api import decode_hidden
d = np.load("/root/repo/data/workloads.npz")
eng = get_engine(); c = make_consts(sd.NetworkConfig(), sd.default_filter_bank())
w = torch.from_numpy(np.load("/root/repo/data/w_fix.npz")["w_fix"]).cuda()
for n in (16, 300, 1250):
    x = torch.from_numpy(d["c3_images"][:n].reshape(n, -1).copy()).cuda()
    outs = {}
    for mode in (5, 3):
        eng.lib.snn_set_hidden_resident(mode)
        o = eng.infer(c, x, w, raster=True); eng.stream.synchronize()
        r = o["raster"].cpu().numpy(); tb = o["tile_base"].cpu().numpy(); tp = o["tile_pos"].cpu().numpy(); nt = o["n_tiles"].cpu().numpy()
        H = [decode_hidden(r, int(tb[i]), tp[i], int(nt[i]), c.n_steps) for i in range(n)]
        outs[mode] = (H, o["counts"].cpu().numpy(), int(o["hidden_redo"].item()))
    eng.lib.snn_set_hidden_resident(1)
    bad = [i for i in range(n) if not np.array_equal(outs[5][0][i], outs[3][0][i])]
    print(n, "redo", outs[5][2], "images with different hidden rasters:", len(bad), bad[:5], "counts equal", np.array_equal(outs[5][1], outs[3][1]))
    if bad:
        i = bad[0]; diff = np.argwhere(outs[5][0][i] != outs[3][0][i]); print("  first diffs (step, neuron):", diff[:5].tolist(), "gb", outs[5][0][i][tuple(diff[0])], "f64", outs[3][0][i][tuple(diff[0])])
