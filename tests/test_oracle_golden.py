"""Pin the oracle (oracle/snn_oracle.py) to vectors produced by the reference
itself (oracle/gen_golden.py -> tests/golden/reference_golden.npz, data/*.npz).

Integer outputs (spikes, counts) must be identical.  Float outputs are
bit-identical on a machine whose BLAS matches the one the goldens were made
with; elsewhere the tolerances below (summation order of dgemm/dgemv/ddot
only) apply.
"""
import dataclasses
import hashlib

import numpy as np
import pytest


def test_input_table(oracle, oparams, golden):
    spk, ctab = oracle.input_table(oparams)
    assert np.array_equal(spk, golden["table_dt1_spk"])
    assert np.array_equal(ctab, golden["table_dt1_c"])   # pure elementwise: bit-exact anywhere


def test_input_table_dt01(oracle, golden):
    spk, ctab = oracle.input_table(oracle.Params(dt=1e-4))
    assert hashlib.sha256(ctab.tobytes()).digest() == golden["table_dt01_sha"].tobytes()
    assert np.array_equal(spk.sum(axis=0), golden["table_dt01_spkcount"])
    assert np.array_equal(ctab[::97], golden["table_dt01_c_rows"])


def test_hidden_currents(oracle, oparams, golden, workloads):
    cur = oracle.hidden_currents(workloads["c3_images"][0], oparams)
    want = golden["c3_0_hidden_currents"]
    assert cur.shape == (100, 8112)
    np.testing.assert_allclose(cur, want, rtol=1e-13, atol=1e-24)


def test_counts_prefix(oracle, oparams, golden, workloads, wfix):
    ctab = oracle.input_table(oparams)[1]
    got = np.stack([oracle.simulate(x, wfix["w_fix"], oparams, ctab=ctab)["counts"]
                    for x in workloads["c3_images"][:24]])
    assert np.array_equal(got, golden["c3_counts_200"][:24])


def test_counts_random_weights(oracle, oparams, golden, workloads):
    ctab = oracle.input_table(oparams)[1]
    got = np.stack([oracle.simulate(x, golden["w_rand"], oparams, ctab=ctab)["counts"]
                    for x in workloads["c3_images"][:8]])
    assert np.array_equal(got, golden["c3_counts_wrand_40"][:8])
    p0 = dataclasses.replace(oparams, inh=0.0)
    got = np.stack([oracle.simulate(x, golden["w_rand"], p0, ctab=ctab)["counts"]
                    for x in workloads["c3_images"][:6]])
    assert np.array_equal(got, golden["c3_counts_wrand_noinh_20"][:6])


def test_counts_t75(oracle, golden, workloads, wfix):
    p = oracle.Params(t=0.075)
    ctab = oracle.input_table(p)[1]
    got = np.stack([oracle.simulate(x, wfix["w_fix"], p, ctab=ctab)["counts"] for x in workloads["c4_images"][:12]])
    assert np.array_equal(got, golden["c4_counts_t75_100"][:12])


@pytest.mark.parametrize("k", [0, 3])
def test_rasters(oracle, oparams, golden, workloads, wfix, k):
    rec = oracle.simulate(workloads["c3_images"][k], wfix["w_fix"], oparams, record=True)
    want = np.unpackbits(golden[f"rec{k}_hidden_bits"], axis=1)[:, :8112].astype(bool)
    assert np.array_equal(rec["hidden"], want)
    assert np.array_equal(rec["out"], golden[f"rec{k}_out"])


def test_training_trajectory_prefix(oracle, oparams, workloads, wfix):
    order = workloads["c2_order"]
    imgs, labs = workloads["c2_images"][order], workloads["c2_labels"][order]
    snaps = {}
    w, counts = oracle.train_epoch(imgs[:20], labs[:20], np.zeros((8112, 10)), oparams,
                                   on_image=lambda i, W: snaps.__setitem__(i + 1, W.copy()))
    assert np.array_equal(counts, wfix["train_counts"][:20])
    for n in (1, 2, 5, 20):
        ref = wfix[f"w_after_{n}"]
        assert np.abs(snaps[n] - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1e-300)


def test_teacher_forced_update(oracle, oparams, golden, workloads, wfix):
    order = workloads["c2_order"]
    j = order[5]
    w0 = wfix["w_after_5"]
    w1, counts, dw = oracle.train_image(workloads["c2_images"][j], int(workloads["c2_labels"][j]), w0, oparams)
    want = golden["tf_w_after_5_dw"]
    assert np.array_equal(counts, golden["tf_w_after_5_counts"])
    assert np.abs(dw - want).max() <= 1e-9 * np.abs(want).max()


def test_pairwise10_matches_numpy_sum(oracle):
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, size=(5000, 10)) * 10.0 ** rng.integers(-8, 8, size=(5000, 10))
    for row in x:
        assert oracle.pairwise10(list(map(float, row))) == float(row.sum())


def test_desired_steps(oracle):
    assert oracle.desired_steps(oracle.Params(dt=1e-4)).tolist()[:2] == [34, 69]
    assert len(oracle.desired_steps(oracle.Params(dt=1e-4))) == 28
    assert oracle.desired_steps(oracle.Params(rate=0.0)).size == 0


def test_default_inhibition(oracle, oparams):
    assert oparams.inhibition == -5.092904083446687e-08


def test_toy_two_class_convergence(oracle, oparams, toy):
    """test_normad.py:236-247 on the oracle: per-epoch errors and weights."""
    w = np.zeros((8112, 10))
    errors = []
    for order in toy["toy_orders"]:
        labs = toy["toy_labels"][order]
        w, counts = oracle.train_epoch(toy["toy_images"][order], labs, w, oparams)
        errors.append(int(sum(oracle.classify(c) != l for c, l in zip(counts, labs))))
    assert errors == toy["toy_errors"].tolist() and errors[-1] == 0
    np.testing.assert_allclose(w, toy["toy_w"], rtol=1e-10, atol=1e-22)


def test_lateral_inhibition_corpus(oracle, oparams, toy):
    """test_network.py:244-258 on the oracle: counts with and without inhibition."""
    no_inh = dataclasses.replace(oparams, inh=0.0)
    ctab = oracle.input_table(oparams)[1]
    for k, im in enumerate(toy["inh_images"]):
        assert np.array_equal(oracle.simulate(im, toy["inh_w"], oparams, ctab=ctab)["counts"], toy["inh_with"][k])
        assert np.array_equal(oracle.simulate(im, toy["inh_w"], no_inh, ctab=ctab)["counts"], toy["inh_without"][k])
