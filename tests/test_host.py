"""Host-side logic of the API mirror (no GPU): config types and validation
mirror the reference (spikedigits), constants derivation, raster decoding,
sharding bounds, and the install() shim."""
import dataclasses
import math
import sys

import numpy as np
import pytest


def test_sizes(sd):
    assert sd.N_HIDDEN == 8112 and sd.parameter_count() == 81_120


def test_config_validation(sd):
    with pytest.raises(ValueError):
        sd.NetworkConfig(t=0.1, dt=3e-4)
    with pytest.raises(ValueError):
        sd.NetworkConfig(desired_rate=400.0)
    with pytest.raises(ValueError):
        sd.NetworkConfig(inhibition_weight=1e-9)
    with pytest.raises(ValueError):
        sd.NetworkConfig(encoding=sd.EncodingParams(i_0=2000e-12))
    cfg = sd.NetworkConfig()
    assert cfg.inhibition_weight == -sd.single_synapse_rate_weight(cfg.output_lif, cfg.desired_rate)
    assert cfg.inhibition_weight == -5.092904083446687e-08
    assert sd.NetworkConfig(desired_rate=0.0).inhibition_weight == 0.0
    with pytest.raises(ValueError):
        sd.LifParams(capacitance=0)
    with pytest.raises(ValueError):
        sd.LearnConfig(learning_rate=0)


def test_filter_bank_matches_reference_golden(sd, oracle):
    assert np.array_equal(sd.default_filter_bank().weighted, oracle._sobel_bank())
    with pytest.raises(ValueError):
        sd.FilterBank(kernels=np.zeros((11, 3, 3)), gains=np.ones(11))
    with pytest.raises(ValueError):
        sd.FilterBank(kernels=np.full((12, 3, 3), np.nan), gains=np.ones(12))


def test_desired_train(sd):
    steps = sd.desired_spike_train(0.100, 1e-4, 285.0)
    assert len(steps) == 28 and steps[0] == 34
    assert sd.desired_spike_train(0.010, 1e-3, 100.0).tolist() == [9]
    assert sd.desired_spike_train(0.1, 1e-3, 0.0).size == 0
    with pytest.raises(ValueError):
        sd.desired_spike_train(0.1, 1e-3, 350.0)


def test_classify(sd):
    assert sd.classify(np.array([5, 5, 0, 0, 0, 0, 0, 0, 0, 0])) == 0
    assert sd.classify(np.zeros(10, dtype=int)) == 0
    c = np.zeros(10, dtype=np.int64)
    c[7] = 28
    assert sd.classify(c) == 7
    with pytest.raises(ValueError):
        sd.classify(np.zeros(9))


def test_pixel_validation(sd):
    assert sd.as_pixel_image(np.arange(784) % 256).shape == (28, 28)
    for bad in (np.zeros((27, 28)), np.full((28, 28), 0.5), np.full((28, 28), 300), np.full((28, 28), np.nan)):
        with pytest.raises(ValueError):
            sd.as_pixel_image(bad)
    assert sd.as_pixel_batch(np.zeros((3, 784))).shape == (3, 28, 28)
    with pytest.raises(ValueError):
        sd.as_pixel_batch(np.zeros(784))
    with pytest.raises(ValueError):
        sd.check_weights(np.full((2, 2), np.inf))


def test_consts_follow_reference_expressions(sd):
    from paper_1711_03637_b200.engine import make_consts
    cfg = sd.NetworkConfig()
    c = make_consts(cfg, sd.default_filter_bank(), sd.LearnConfig())
    assert c.n_steps == 100 and c.desired_period == 4
    assert c.lif_hid.beta == 3166666.6666666665
    assert c.lif_hid.refr == 3e-3 / 1e-3
    assert c.decay_slow == math.exp(-1e-3 / 5e-3) == 0.8187307530779818
    assert c.decay_fast == 0.44932896411722156
    assert c.decay_learn == 0.36787944117144233
    assert c.inhibition == cfg.inhibition_weight
    c01 = make_consts(dataclasses.replace(cfg, dt=1e-4), sd.default_filter_bank())
    assert c01.lif_out.beta == 331666.6666666667 and c01.desired_period == 35 and c01.n_steps == 1000
    taps = np.ctypeslib.as_array(c.taps)
    assert np.array_equal(taps, sd.default_filter_bank().weighted.reshape(12, 9))
    with pytest.raises(ValueError), np.errstate(over="ignore"):  # taps overflow to inf: rejected
        make_consts(cfg, sd.FilterBank(kernels=np.full((12, 3, 3), 1e306), gains=np.full(12, 1e3)))


def test_decode_hidden_roundtrip():
    from paper_1711_03637_b200.api import decode_hidden
    rng = np.random.default_rng(0)
    N, tb = 20, 5
    want = np.zeros((N, 8112), dtype=bool)
    active = np.sort(rng.choice(676, size=70, replace=False))
    nt = 3
    nch = -(-N // 8)
    raster = np.zeros((tb + nt) * nch * 512, dtype=np.uint8)
    blk = raster[tb * nch * 512:].reshape(nch, nt, 2, 32, 8)
    tpos = np.full((22, 32), -1, dtype=np.int16)
    for slot, p in enumerate(active):
        t, lane = divmod(slot, 32)
        tpos[t, lane] = p
        m = rng.integers(0, 4096, size=N) & rng.integers(0, 4096, size=N)
        for s_ in range(N):
            blk[s_ // 8, t, 0, lane, s_ % 8] = m[s_] & 0x3F
            blk[s_ // 8, t, 1, lane, s_ % 8] = m[s_] >> 6
        for f in range(12):
            want[:, p * 12 + f] = (m >> f) & 1
    got = decode_hidden(raster, tb, tpos, nt, N)
    assert np.array_equal(got, want)


def test_shard_bounds_match_array_split():
    from paper_1711_03637_b200.distributed import shard_bounds
    for n in (0, 1, 7, 10_000, 10_001):
        for w in (1, 2, 3, 8):
            idx = np.array_split(np.arange(n), w)
            assert [(int(a[0]), int(a[-1]) + 1) if len(a) else None for a in idx] == \
                [(a, b) if b > a else None for a, b in shard_bounds(n, w)]


def test_shim_install_rebinds_reference():
    pytest.importorskip("sklearn")
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        sdr = pytest.importorskip("spikedigits")
    finally:
        sys.path.pop(0)
    import spikedigits.evaluate as ev
    import spikedigits.normad as nm

    from paper_1711_03637_b200 import api, shim
    orig = ev.batch_counts
    n = shim.install()
    try:
        assert n >= 10
        assert ev.batch_counts is api.batch_counts
        assert nm.train_epoch is api.train_epoch
        assert sdr.forward_pass is api.forward_pass
        assert api._NUMERIC_ERROR is nm.NumericFailureError
        import spikedigits.cli as cli
        import spikedigits.preprocess as rpre
        from paper_1711_03637_b200 import preprocess as gpre
        assert cli.preprocess_pipeline is gpre.preprocess_pipeline
        assert gpre._BLANK_ERROR is rpre.BlankDrawingError
    finally:
        shim.uninstall()
    assert ev.batch_counts is orig
    assert gpre._BLANK_ERROR is gpre.BlankDrawingError
