"""GPU parity, widened (round 2): per-neuron hidden spike counts on 1,000
reference images, all 10,000 config-5 eval images, the near-tie detector, the
level-0 liveness guard, serving-graph lifetime, off-path canvases."""
import dataclasses
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_1711_03637_b200 import _native  # noqa: E402
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def cfg(sd):
    return sd.NetworkConfig()


@pytest.fixture(scope="module")
def bank(sd):
    return sd.default_filter_bank()


def _hidden_counts_first(eng, c, imgs, w):
    """Per-neuron hidden spike counts and first spike steps of a batch through
    one snn_infer call with the compact raster (decoded on the host)."""
    from paper_1711_03637_b200.api import decode_hidden
    d_img = torch.from_numpy(imgs.reshape(len(imgs), -1).copy()).to(eng.device)
    d_w = torch.from_numpy(w.copy()).to(eng.device)
    out = eng.infer(c, d_img, d_w, raster=True)
    eng.stream.synchronize()
    raster = out["raster"].cpu().numpy()
    tpos, nt, tb = out["tile_pos"].cpu().numpy(), out["n_tiles"].cpu().numpy(), out["tile_base"].cpu().numpy()
    cnt = np.zeros((len(imgs), 8112), dtype=np.int64)
    first = np.full((len(imgs), 8112), -1, dtype=np.int64)
    for i in range(len(imgs)):
        h = decode_hidden(raster, int(tb[i]), tpos[i], int(nt[i]), c.n_steps)
        cnt[i] = h.sum(axis=0)
        any_ = h.any(axis=0)
        first[i, any_] = np.argmax(h[:, any_], axis=0)
    return cnt, first, out["counts"].cpu().numpy()


def test_hidden_per_neuron_counts_1000_reference_images(sd, cfg, bank, workloads, wfix):
    """north_star: identical spike counts PER NEURON.  The reference's own
    forward_pass on every 10th config-3 image (1,000 images, 8,112 neurons
    each; oracle/gen_hidden_counts.py): hidden spike counts and first spike
    steps of every neuron, and the output counts, through the GPU raster."""
    from paper_1711_03637_b200.engine import get_engine, make_consts
    g = np.load(os.path.join(GOLD, "c3_hidden_counts_reference.npz"))
    imgs = workloads["c3_images"][g["idx"]]
    cnt, first, out = _hidden_counts_first(get_engine(), make_consts(cfg, bank), imgs, wfix["w_fix"])
    same = (cnt == g["hidden_counts"]).all(axis=1)
    print(f"per-neuron hidden counts identical on {same.mean():.6f} of 1,000 images "
          f"({int(g['hidden_counts'].astype(np.int64).sum())} reference spikes)")
    assert same.all()
    assert np.array_equal(first, g["first_spike"].astype(np.int64))
    assert np.array_equal(out, g["output_counts"])
    # and through the public forward_pass for a few of them
    for i in (0, 499, 999):
        rec = sd.forward_pass(imgs[i], wfix["w_fix"], bank, cfg)
        assert np.array_equal([len(x) for x in rec.hidden_spikes], g["hidden_counts"][i])


def test_c5_eval_all_10000_vs_reference(sd, cfg, bank):
    """The reference's batch_counts on all 10,000 config-5 eval images under
    its own weights after the 60,000-image pass (oracle/gen_c5_eval.py)."""
    d5 = np.load(os.path.join(ROOT, "data", "c5_workload.npz"))
    w = np.load(os.path.join(GOLD, "c5_reference.npz"))["w_after_60000"]
    want = np.load(os.path.join(GOLD, "c5_eval_reference.npz"))["eval_counts"]
    got = sd.batch_counts(d5["eval_images"], w, bank, cfg)
    assert np.array_equal(got, want)


def test_near_ties_none_on_the_workloads(sd, cfg, bank, workloads, wfix):
    """The near-tie detector (snn_infer_out_t.near_ties) on all 10,000 config-3
    images: no output step lies within the rounding bound of the reordered
    c_hidden @ W sum, i.e. the identical counts are guaranteed, not observed.
    Counts with the detector on equal counts without it."""
    from paper_1711_03637_b200.engine import get_engine, make_consts
    eng, c = get_engine(), make_consts(cfg, bank)
    imgs = workloads["c3_images"]
    d_img = torch.from_numpy(imgs.reshape(len(imgs), -1).copy()).to(eng.device)
    d_w = torch.from_numpy(wfix["w_fix"].copy()).to(eng.device)
    out = eng.infer(c, d_img, d_w, ties=True)
    eng.stream.synchronize()
    ties = out["near_ties"].cpu().numpy()
    ref = np.load(os.path.join(GOLD, "c3_counts_reference.npz"))["counts"]
    assert np.array_equal(out["counts"].cpu().numpy(), ref)
    print("near ties on 10,000 c3 images:", int(ties.sum()))
    assert int(ties.sum()) == 0


def test_near_tie_detector_flags_a_constructed_tie(sd, cfg, bank, workloads, wfix):
    """A weight scale bisected (on the GPU path itself) to the point where
    output 0 first reaches threshold: at the crossing scale the decisive step
    has |v - V_T| at rounding level and must be flagged; at 0.98x of it the
    neuron stays silent and nothing is flagged."""
    from paper_1711_03637_b200.engine import get_engine, make_consts
    eng, c = get_engine(), make_consts(cfg, bank)
    img = workloads["c3_images"][:1].reshape(1, -1).copy()
    d_img = torch.from_numpy(img).to(eng.device)
    u = np.abs(wfix["w_fix"][:, 0])

    def run(scale):
        w = np.zeros((8112, 10))
        w[:, 0] = u * scale
        o = eng.infer(c, d_img, torch.from_numpy(w).to(eng.device), ties=True)
        eng.stream.synchronize()
        return int(o["counts"][0, 0].item()), int(o["near_ties"][0].item())

    lo, hi = 0.0, 1.0
    while run(hi)[0] == 0:
        hi *= 2.0
    for _ in range(200):  # down to adjacent doubles
        mid = 0.5 * (lo + hi)
        if mid in (lo, hi):
            break
        if run(mid)[0] == 0:
            lo = mid
        else:
            hi = mid
    cnt_hi, ties_hi = run(hi)
    cnt_lo, ties_lo = run(lo)
    assert cnt_lo == 0 and cnt_hi >= 1
    assert ties_hi >= 1 and ties_lo >= 1  # both sides of the crossing are within the bound
    cnt_far, ties_far = run(0.98 * lo)
    assert cnt_far == 0 and ties_far == 0


def test_level0_spiking_simulates_every_window(sd, cfg, bank, wfix, workloads, oracle):
    """i_0 just above the rheobase (accepted by the reference's rel_tol 1e-9,
    network.py:133-136): pixel level 0 spikes in a 500 ms trial, so all-zero
    windows receive current; with an all-positive bank they fire.  k_prep
    then simulates every window: counts and the hidden raster of a blank and a
    digit image against the oracle."""
    from paper_1711_03637_b200.params import min_spiking_current
    rh = min_spiking_current(cfg.input_lif)
    c_ = dataclasses.replace(cfg, encoding=dataclasses.replace(cfg.encoding, i_0=rh * (1 + 9e-10)), t=0.5)
    b = sd.FilterBank(kernels=np.ones((12, 3, 3)), gains=np.full(12, 3e-9))
    p = oracle.params_from_reference(c_, b)
    assert (oracle.input_table(p)[1][:, 0] != 0).any()   # level 0 does spike
    imgs = np.stack([np.zeros((28, 28), np.uint8), workloads["c3_images"][0]])
    w = wfix["w_fix"]
    recs = [oracle.simulate(x, w, p, record=True) for x in imgs]
    assert recs[0]["hidden"].sum() > 0                     # the blank image's windows fire
    got = sd.batch_counts(imgs, w, b, c_)
    assert np.array_equal(got, np.stack([r["counts"] for r in recs]))
    rec = sd.forward_pass(imgs[0], w, b, c_)
    hm = np.zeros_like(recs[0]["hidden"])
    for k, steps in enumerate(rec.hidden_spikes):
        hm[steps, k] = True
    assert np.array_equal(hm, recs[0]["hidden"])


def test_serving_graphs_bounded_and_keep_their_tables(sd, cfg, bank, workloads, wfix):
    """The batch-1 graphs of many (t, dt) configurations: at most MAX_GRAPHS
    are kept, each holds its own input table, and after the table cache has
    evicted a graph's table the graph still gives the batch path's counts."""
    from paper_1711_03637_b200 import engine as E
    eng = E.get_engine()
    img = workloads["c4_images"][3]
    ts = [0.010 + 0.005 * k for k in range(E.MAX_GRAPHS + 6)]
    first = dataclasses.replace(cfg, t=ts[0])
    want0 = sd.batch_counts(img[None], wfix["w_fix"], bank, first)[0]
    assert np.array_equal(sd.run_presentation(img, wfix["w_fix"], bank, first), want0)
    for t in ts[1:E.MAX_TABLES + 2]:   # evicts the first config's table from the table cache
        sd.run_presentation(img, wfix["w_fix"], bank, dataclasses.replace(cfg, t=t))
    assert len(eng._tables) <= E.MAX_TABLES
    torch.cuda.empty_cache()
    junk = [torch.full((1 << 20,), 7.0, dtype=torch.float64, device=eng.device) for _ in range(8)]
    assert np.array_equal(sd.run_presentation(img, wfix["w_fix"], bank, first), want0)
    del junk
    for t in ts:
        c_ = dataclasses.replace(cfg, t=t)
        assert np.array_equal(sd.run_presentation(img, wfix["w_fix"], bank, c_),
                              sd.batch_counts(img[None], wfix["w_fix"], bank, c_)[0])
    assert len(eng._graphs) <= E.MAX_GRAPHS
    assert all("ctab" in g for g in eng._graphs.values())


def test_canvases_off_the_uint8_path_match_reference(sd):
    """float / int16 / bool canvases, fractional thresholds and canvases over
    1024 px (cropped to the ink on the host) against the reference's own
    outputs (oracle/gen_canvases_extra.py); an ink extent over 1024 px is
    rejected with ValueError."""
    z = np.load(os.path.join(GOLD, "canvases_extra.npz"))
    k = 0
    while f"canvas{k}" in z:
        thr = float(z[f"threshold{k}"])
        thr = int(thr) if thr.is_integer() else thr
        assert np.array_equal(sd.preprocess_pipeline(z[f"canvas{k}"], thr), z[f"out{k}"]), k
        k += 1
    assert k == 6
    big = np.zeros((1200, 1200), dtype=np.uint8)
    big[10:1190, 600:605] = 255
    with pytest.raises(ValueError):
        sd.preprocess_pipeline(big)


def test_two_engines_one_process(sd, cfg, bank, workloads, wfix):
    """Two Engine objects (own streams, workspaces and graphs) used from two
    threads at once give the single-engine results; the per-device state
    (function attributes, occupancy, knobs) of the library is shared by both
    on this device."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_1711_03637_b200.engine import Engine, make_consts
    c = make_consts(cfg, bank)
    imgs = workloads["c3_images"][:256]
    want = sd.batch_counts(imgs, wfix["w_fix"], bank, cfg)
    engs = [Engine("cuda:0"), Engine("cuda:0")]

    def go(e):
        d_img = torch.from_numpy(imgs.reshape(len(imgs), -1).copy()).to(e.device)
        d_w = torch.from_numpy(wfix["w_fix"].copy()).to(e.device)
        r = [e.infer(c, d_img, d_w)["counts"] for _ in range(4)]
        e.stream.synchronize()
        return [x.cpu().numpy() for x in r]

    with ThreadPoolExecutor(2) as ex:
        res = list(ex.map(go, engs))
    for r in res:
        for x in r:
            assert np.array_equal(x, want)


def test_guard_band_hidden_kernel_bit_identical(sd, cfg, bank, workloads, wfix):
    """The guard-band hidden layer (float32 pairs + float64 redo of the flagged
    windows, hidden_gb.cuh) against the float64 kernel (snn_set_hidden_resident
    (3)): the compact hidden raster of all 10,000 config-3 images byte for
    byte, the counts, a 100-image NormAD epoch bit for bit, and the redo
    fraction reported by snn_infer_out_t.hidden_redo."""
    from paper_1711_03637_b200.engine import get_engine, make_consts
    eng, c = get_engine(), make_consts(cfg, bank)
    n = len(workloads["c3_images"])
    imgs = torch.from_numpy(workloads["c3_images"].reshape(n, -1).copy()).to(eng.device)
    w = torch.from_numpy(wfix["w_fix"].copy()).to(eng.device)
    res = {}
    for mode in (1, 3):
        eng.lib.snn_set_hidden_resident(mode)
        try:
            o = eng.infer(c, imgs, w, raster=True)
            eng.stream.synchronize()
            nb = int(o["tile_base"][n].item()) * (-(-c.n_steps // 8)) * 512
            res[mode] = (o["raster"][:nb].cpu().numpy(), o["counts"].cpu().numpy(), int(o["hidden_redo"].item()))
        finally:
            eng.lib.snn_set_hidden_resident(1)
    assert np.array_equal(res[1][0], res[3][0])
    assert np.array_equal(res[1][1], res[3][1])
    redo = res[1][2]
    print(f"guard band: {redo} windows re-simulated in float64 (of 3,571,517 active)")
    assert 0 < redo < 0.25 * 3_571_517
    order = workloads["c2_order"][:100]
    ims, labs = workloads["c2_images"][order], workloads["c2_labels"][order]
    out = []
    # small batches: the default takes the float64 kernel (no redo); mode 5
    # forces the guard band there too -- same raster
    small = imgs[:16]
    o = eng.infer(c, small, w, raster=True)
    eng.stream.synchronize()
    assert int(o["hidden_redo"].item()) == 0
    from paper_1711_03637_b200.api import decode_hidden
    rs = []
    for mode in (5, 3):  # decoded per image: raster bytes of padding lanes are never written
        eng.lib.snn_set_hidden_resident(mode)
        try:
            o = eng.infer(c, small, w, raster=True)
            eng.stream.synchronize()
            r, tb, tp, nt = (o[k].cpu().numpy() for k in ("raster", "tile_base", "tile_pos", "n_tiles"))
            rs.append((np.stack([decode_hidden(r, int(tb[i]), tp[i], int(nt[i]), c.n_steps) for i in range(16)]),
                       o["counts"].cpu().numpy()))
        finally:
            eng.lib.snn_set_hidden_resident(1)
    assert rs[0][0].any()
    assert np.array_equal(rs[0][0], rs[1][0]) and np.array_equal(rs[0][1], rs[1][1])
    for mode in (5, 3):  # 5: the guard band also for the 64-image first chunk
        eng.lib.snn_set_hidden_resident(mode)
        try:
            out.append(sd.train_epoch(ims, labs, sd.zero_weights(), bank, cfg, sd.LearnConfig())[0])
        finally:
            eng.lib.snn_set_hidden_resident(1)
    assert np.array_equal(out[0], out[1])


def test_speculative_normad_bit_identical(sd, cfg, bank, workloads):
    """The speculative-scan NormAD kernel (snn_set_normad_cluster(4), the
    default; normad_spec.cuh) runs image i+1's output scan on the sums of the weights
    before image i's update and proves it (or redoes it): its weights and
    per-image counts equal the plain cluster kernel's bit for bit, and
    d_status[3] counts the redone scans."""
    from paper_1711_03637_b200.engine import get_engine, make_consts
    eng = get_engine()
    c = make_consts(cfg, bank, sd.LearnConfig())
    n = 300
    order = workloads["c2_order"][:n]
    imgs = torch.from_numpy(workloads["c2_images"][order].reshape(n, -1).copy()).to(eng.device)
    labs = torch.from_numpy(workloads["c2_labels"][order].astype(np.uint8)).to(eng.device)
    res = {}
    for mode in (3, 4):
        eng.lib.snn_set_normad_cluster(mode)
        try:
            w = torch.zeros((8112, 10), dtype=torch.float64, device=eng.device)
            cnt, status = eng.train(c, imgs, labs, w)
            eng.stream.synchronize()
            res[mode] = (w.cpu().numpy(), cnt.cpu().numpy(), status.cpu().numpy())
        finally:
            eng.lib.snn_set_normad_cluster(_native.NORMAD_DEFAULT)
    assert np.array_equal(res[3][0], res[4][0])
    assert np.array_equal(res[3][1], res[4][1])
    assert res[4][2][0] == 0 and res[4][2][2] == n
    print(f"speculative scans redone: {res[4][2][3]} of {n - 1}")
    assert 0 <= res[4][2][3] < n


def test_output_dist_bit_identical(sd, cfg, bank, workloads, wfix):
    """The lane-distributed output layer (k_output_dist, batches >= 256) and
    the replicated-trace one (snn_set_output_dist(0)): counts, ff, v_out and
    the output raster of 300 config-3 images bit for bit."""
    from paper_1711_03637_b200.engine import get_engine, make_consts
    eng = get_engine()
    c = make_consts(cfg, bank)
    n = 300
    imgs = torch.from_numpy(workloads["c3_images"][:n].reshape(n, -1).copy()).to(eng.device)
    w = torch.from_numpy(wfix["w_fix"].copy()).to(eng.device)
    res = []
    for mode in (1, 0):
        eng.lib.snn_set_output_dist(mode)
        try:
            o = eng.infer(c, imgs, w, trace=True)
            o2 = eng.infer(c, imgs, w, raster=True)
            eng.stream.synchronize()
            res.append([o[k].cpu().numpy() for k in ("counts", "ff", "v_out")] + [o2["out_raster"].cpu().numpy()])
        finally:
            eng.lib.snn_set_output_dist(1)
    assert res[0][0].sum() > 0
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)


def test_guard_band_long_trial_chunked_redo(sd, cfg, bank, workloads, wfix):
    """T = 150 ms (N = 150 > 108 steps: the float64 redo streams the table in
    chunks, k_hidden_fix, instead of holding it in shared memory): the guard
    band against the float64 ring kernel on 1,000 config-3 images -- counts
    and the decoded hidden rasters of 40 of them."""
    from paper_1711_03637_b200.api import decode_hidden
    from paper_1711_03637_b200.engine import get_engine, make_consts
    eng = get_engine()
    c = make_consts(dataclasses.replace(cfg, t=0.15), bank)
    assert c.n_steps == 150
    n = 1000
    imgs = torch.from_numpy(workloads["c3_images"][:n].reshape(n, -1).copy()).to(eng.device)
    w = torch.from_numpy(wfix["w_fix"].copy()).to(eng.device)
    res = {}
    for mode in (1, 3):
        eng.lib.snn_set_hidden_resident(mode)
        try:
            o = eng.infer(c, imgs, w, raster=True)
            eng.stream.synchronize()
            r, tb, tp, nt = (o[k].cpu().numpy() for k in ("raster", "tile_base", "tile_pos", "n_tiles"))
            dec = np.stack([decode_hidden(r, int(tb[i]), tp[i], int(nt[i]), c.n_steps) for i in range(0, n, 25)])
            res[mode] = (o["counts"].cpu().numpy(), dec, int(o["hidden_redo"].item()))
        finally:
            eng.lib.snn_set_hidden_resident(1)
    assert res[1][2] > 0  # the guard band ran and flagged some windows
    assert res[1][1].any()
    assert np.array_equal(res[1][0], res[3][0])
    assert np.array_equal(res[1][1], res[3][1])


def test_sharded_batch_counts_two_ranks_one_gpu():
    """distributed.sharded_batch_counts (the multi-GPU e2e path of bench.py)
    with two ranks sharing one GPU over gloo: its counts equal batch_counts'
    (scripts/sharded_check.py under torchrun)."""
    import subprocess
    import sys
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541",
                        os.path.join(ROOT, "scripts", "sharded_check.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("sharded == batch_counts: True") == 2
