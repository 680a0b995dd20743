"""CPU oracle for the SNN inference + NormAD hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1711_03637_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or the timed CPU reference), never as the product path.

It restates, in float64 numpy, the algorithm of the reference package
``spikedigits`` (``/root/reference/pkg/src/spikedigits``), keeping the
reference's operation order so that, on the same machine and BLAS, results
are bit-identical to the reference.  That claim is pinned by
``tests/test_oracle_golden.py`` against vectors produced by the reference
itself (``oracle/gen_golden.py`` -> ``tests/golden/*.npz``).

Citations are ``file:line`` relative to ``/root/reference/pkg/src/spikedigits``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

SIDE = 28          # network.py:36
FMAP = 26          # network.py:37
NFILT = 12         # network.py:38
NPIX = SIDE * SIDE
NHID = NFILT * FMAP * FMAP   # 8112, network.py:40
NOUT = 10          # network.py:41
TAU1 = 5e-3        # neurons.py:19
TAU2 = 1.25e-3     # neurons.py:20
TAU_L = 1e-3       # normad.py:30


@dataclass(frozen=True)
class Lif:
    """One population's constants (neurons.py:23-37), SI units."""

    C: float = 300e-12
    g: float = 30e-9
    el: float = -70e-3
    vt: float = 20e-3
    tref: float = 3e-3

    def beta(self, dt: float) -> float:
        # neurons.py:118 -- RK2 collapsed factor, same expression order
        return dt * (2.0 - self.g * dt / self.C) / (2.0 * self.C)


def _sobel_bank(drive: float = 15e-9) -> np.ndarray:
    """Weighted 12x3x3 filter bank (filters.py:22-31, :63-88)."""
    h = [[1, 2, 1], [0, 0, 0], [-1, -2, -1]]
    v = [[1, 0, -1], [2, 0, -2], [1, 0, -1]]
    d = [[2, 1, 0], [1, 0, -1], [0, -1, -2]]
    ad = [[0, 1, 2], [-1, 0, 1], [-2, -1, 0]]
    corners = []
    for r0, c0 in ((0, 0), (0, 1), (1, 0), (1, 1)):
        k = np.full((3, 3), -4.0)
        k[r0:r0 + 2, c0:c0 + 2] = 5.0
        corners.append(k)
    k = np.array([h, v, d, ad] + [np.negative(x) for x in (h, v, d, ad)], dtype=np.float64)
    k = np.concatenate([k, np.array(corners)], axis=0)
    gains = drive / np.clip(k, 0.0, None).sum(axis=(1, 2))
    return k * gains[:, None, None]


@dataclass(frozen=True)
class Params:
    """Everything the hot path reads from NetworkConfig / FilterBank."""

    t: float = 0.100
    dt: float = 1e-3
    rate: float = 285.0
    inh: float | None = None
    i0: float = 2700e-12
    ip: float = 101.2e-12
    lif_in: Lif = Lif()
    lif_hid: Lif = Lif()
    lif_out: Lif = Lif()
    taps: np.ndarray = field(default_factory=_sobel_bank, compare=False)

    @property
    def n_steps(self) -> int:
        return int(round(self.t / self.dt))     # network.py:148-150

    @property
    def inhibition(self) -> float:
        """network.py:137-144 (single_synapse_rate_weight at :80-101)."""
        if self.inh is not None:
            return float(self.inh)
        if self.rate <= 0:
            return 0.0
        o = self.lif_out
        charge = 1.0 / self.rate - o.tref
        tau_m = o.C / o.g
        i_need = (o.g * (o.vt - o.el)) / -math.expm1(-charge / tau_m)
        return -(i_need / (self.rate * (TAU1 - TAU2)))


def params_from_reference(cfg, bank) -> Params:
    """Build oracle Params from reference (or API-mirror) objects."""
    def lif(x):
        return Lif(x.capacitance, x.leak_conductance, x.rest_potential, x.threshold, x.refractory)
    return Params(t=cfg.t, dt=cfg.dt, rate=cfg.desired_rate, inh=cfg.inhibition_weight,
                  i0=cfg.encoding.i_0, ip=cfg.encoding.i_p, lif_in=lif(cfg.input_lif),
                  lif_hid=lif(cfg.hidden_lif), lif_out=lif(cfg.output_lif),
                  taps=np.array(bank.weighted, dtype=np.float64))


# ---------------------------------------------------------------- primitives

def _lif_update(v, last, drive, lif: Lif, dt: float, step: int):
    """neurons.py:113-126, elementwise, identical op order (no FMA)."""
    live = step > last + lif.tref / dt
    cand = v + lif.beta(dt) * (drive - lif.g * (v - lif.el))
    cand = np.maximum(cand, lif.el)
    fired = live & (cand >= lif.vt)
    v = np.where(live, np.where(fired, lif.el, cand), v)
    last = np.where(fired, float(step), last)
    return v, last, fired


def _decays(dt: float):
    """neurons.py:148-150 and normad.py:82 (host libm exp, never device exp)."""
    return math.exp(-dt / TAU1), math.exp(-dt / TAU2), math.exp(-dt / TAU_L)


def input_table(p: Params):
    """network.py:224-245: 256 pixel levels simulated once -> (spk, c), (N,256)."""
    n = p.n_steps
    lam1, lam2, _ = _decays(p.dt)
    drive = p.i0 + np.arange(256) * p.ip               # network.py:72-77
    v = np.full(256, p.lif_in.el)
    last = np.full(256, -np.inf)
    a = np.zeros(256)
    b = np.zeros(256)
    spk = np.zeros((n, 256), dtype=bool)
    ctab = np.zeros((n, 256))
    for s in range(n):
        v, last, fired = _lif_update(v, last, drive, p.lif_in, p.dt, s)
        bump = fired.astype(np.float64)
        a = a * lam1 + bump                            # neurons.py:169-171
        b = b * lam2 + bump
        spk[s] = fired
        ctab[s] = a - b
    return spk, ctab


def hidden_currents(image, p: Params, ctab=None) -> np.ndarray:
    """network.py:212-221 + :254-264: (N, 8112) currents, index (r*26+c)*12+f."""
    if ctab is None:
        ctab = input_table(p)[1]
    lev = np.asarray(image, dtype=np.uint8).reshape(SIDE, SIDE)
    cmap = ctab[:, lev.ravel()].reshape(-1, SIDE, SIDE)
    win = sliding_window_view(cmap, (3, 3), axis=(1, 2))           # (N,26,26,3,3)
    rows = np.ascontiguousarray(win).reshape(-1, 9)
    taps = np.ascontiguousarray(np.asarray(p.taps, dtype=np.float64).reshape(NFILT, 9).T)
    return (rows @ taps).reshape(cmap.shape[0], NHID)   # BLAS dgemm, k-ordered FMA chain


def pairwise10(x) -> float:
    """numpy's pairwise add-reduce for 10 float64 (what ``c_out.sum()`` does)."""
    r = ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7]))
    r = r + x[8]
    return r + x[9]


def desired_steps(p: Params) -> np.ndarray:
    """network.py:171-193."""
    if p.rate == 0:
        return np.empty(0, dtype=np.int64)
    period = max(1, int(math.floor(1.0 / (p.rate * p.dt) + 0.5)))
    return np.arange(period - 1, p.n_steps, period, dtype=np.int64)


# ---------------------------------------------------------------- one trial

def simulate(image, W, p: Params, ctab=None, record: bool = False, hook=None):
    """network.py:267-326 (run_presentation) with optional recording.

    Returns dict with ``counts`` (int64[10]); when ``record``: ``hidden``
    (bool[N,8112]), ``out`` (bool[N,10]), ``ff`` (c_hidden@W, [N,10]),
    ``v_out`` ([N,10]) and ``v_hid`` ([N,8112]).
    """
    W = np.asarray(W, dtype=np.float64)
    cur = hidden_currents(image, p, ctab)
    if not np.all(np.isfinite(cur)):
        raise ValueError("hidden currents contain non-finite values")
    n = p.n_steps
    lam1, lam2, _ = _decays(p.dt)
    inh = p.inhibition
    vh = np.full(NHID, p.lif_hid.el)
    lh = np.full(NHID, -np.inf)
    ah = np.zeros(NHID)
    bh = np.zeros(NHID)
    vo = np.full(NOUT, p.lif_out.el)
    lo = np.full(NOUT, -np.inf)
    ao = np.zeros(NOUT)
    bo = np.zeros(NOUT)
    prev = np.zeros(NOUT, dtype=bool)
    counts = np.zeros(NOUT, dtype=np.int64)
    rec = {}
    if record:
        rec = {k: np.zeros(s, dtype=d) for k, s, d in (
            ("hidden", (n, NHID), bool), ("out", (n, NOUT), bool),
            ("ff", (n, NOUT), np.float64), ("v_out", (n, NOUT), np.float64),
            ("v_hid", (n, NHID), np.float64))}
    for s in range(n):
        vh, lh, hf = _lif_update(vh, lh, cur[s], p.lif_hid, p.dt, s)
        bump = hf.astype(np.float64)
        ah = ah * lam1 + bump
        bh = bh * lam2 + bump
        ch = ah - bh
        pb = prev.astype(np.float64)
        ao = ao * lam1 + pb
        bo = bo * lam2 + pb
        co = ao - bo
        ff = ch @ W
        drive = ff + inh * (co.sum() - co)
        vo, lo, of = _lif_update(vo, lo, drive, p.lif_out, p.dt, s)
        prev = of
        counts += of
        if record:
            rec["hidden"][s] = hf
            rec["out"][s] = of
            rec["ff"][s] = ff
            rec["v_out"][s] = vo
            rec["v_hid"][s] = vh
        if hook is not None:
            hook(s, ch, of)
    rec["counts"] = counts
    return rec


class NumericFailure(RuntimeError):
    pass


def train_image(image, label: int, W, p: Params, lr: float = 2e-7, eps: float = 1e-12,
                ctab=None):
    """normad.py:141-162 with the hook of :156-159 (dhat_step :75-84,
    error_signal :87-91, accumulate_update :94-114) and apply_update :117-127.
    Returns (W_new, counts, dW)."""
    n = p.n_steps
    target = np.zeros((n, NOUT), dtype=bool)
    target[desired_steps(p), int(label)] = True
    _, _, lamL = _decays(p.dt)
    scale = p.dt / p.lif_out.C
    dhat = np.zeros(NHID)
    dW = np.zeros((NHID, NOUT))

    def hook(s, ch, of):
        nonlocal dhat
        dhat *= lamL
        dhat += np.asarray(ch, dtype=np.float64) * scale
        err = target[s].astype(np.int8) - of.astype(np.int8)
        idx = np.flatnonzero(err)
        if idx.size == 0:
            return
        nrm = float(np.linalg.norm(dhat))
        if nrm <= eps:
            return
        for l in idx:
            dW[:, l] += dhat * (float(err[l]) * p.dt / nrm)

    counts = simulate(image, W, p, ctab=ctab, hook=hook)["counts"]
    W_new = np.asarray(W, dtype=np.float64) + lr * dW
    if not np.all(np.isfinite(W_new)):
        raise NumericFailure("weight update produced non-finite values")
    return W_new, counts, dW


def train_epoch(images, labels, W, p: Params, lr: float = 2e-7, eps: float = 1e-12,
                on_image=None):
    """normad.py:179-207: sequential online pass.  Returns (W, counts[n,10])."""
    ctab = input_table(p)[1]
    W = np.asarray(W, dtype=np.float64)
    out = np.zeros((len(images), NOUT), dtype=np.int64)
    for i, (img, lab) in enumerate(zip(images, labels)):
        W, out[i], _ = train_image(img, int(lab), W, p, lr, eps, ctab=ctab)
        if on_image is not None:
            on_image(i, W)
    return W, out


def classify(counts) -> int:
    """network.py:349-356 (argmax, ties to the lowest index)."""
    return int(np.argmax(np.asarray(counts)))


# ---------------------------------------------------------------- batch (timed CPU reference)

def _chunk_counts(args):
    images, W, p = args
    ctab = input_table(p)[1]
    return np.stack([simulate(img, W, p, ctab=ctab)["counts"] for img in images]) \
        if len(images) else np.zeros((0, NOUT), dtype=np.int64)


def batch_counts(images, W, p: Params, workers: int = 1) -> np.ndarray:
    """evaluate.py:27-40: data parallel over images, concatenated in order."""
    images = np.asarray(images, dtype=np.uint8).reshape(-1, SIDE, SIDE)
    if len(images) == 0:
        return np.zeros((0, NOUT), dtype=np.int64)
    if workers <= 1 or len(images) < 2 * workers:
        return _chunk_counts((images, W, p))
    import multiprocessing as mp
    chunks = [c for c in np.array_split(images, workers) if len(c)]
    with mp.get_context("fork").Pool(workers) as pool:
        parts = pool.map(_chunk_counts, [(c, W, p) for c in chunks])
    return np.concatenate(parts)
