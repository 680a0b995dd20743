"""Canvas preprocessing (preprocess.py:110-115): the oracle's
restatement (incl. Pillow's fixed-point BILINEAR resampling) pinned to the
reference's outputs on CPU, and the GPU kernel against the same fixtures."""
import numpy as np
import pytest


def test_oracle_matches_reference_fixtures(canvases):
    from oracle import preprocess_oracle as P
    for c, t, want, blank in zip(canvases["list"], canvases["thresholds"], canvases["outputs"], canvases["blank"]):
        if blank:
            with pytest.raises(P.BlankDrawing):
                P.preprocess(c, int(t))
        else:
            assert np.array_equal(P.preprocess(c, int(t)), want)


def test_oracle_resize_matches_pillow():
    """The restated resize against Pillow itself (a dependency of the reference)."""
    Image = pytest.importorskip("PIL.Image")
    from oracle import preprocess_oracle as P
    rng = np.random.default_rng(3)
    for _ in range(60):
        h, w = (int(x) for x in rng.integers(1, 160, 2))
        nh, nw = (int(x) for x in rng.integers(1, 40, 2))
        img = rng.integers(0, 256, (h, w)).astype(np.uint8)
        want = np.asarray(Image.fromarray(img).resize((nw, nh), Image.Resampling.BILINEAR))
        assert np.array_equal(P.resize_bilinear(img, nw, nh), want)


@pytest.mark.gpu
def test_gpu_batch_matches_reference(canvases):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1711_03637_b200 as sd
    imgs, blank = sd.preprocess_batch(canvases["list"], canvases["thresholds"])
    assert np.array_equal(blank, canvases["blank"].astype(bool))
    assert np.array_equal(imgs, canvases["outputs"])


@pytest.mark.gpu
def test_gpu_pipeline_single_and_errors(canvases):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1711_03637_b200 as sd
    for k in (0, 7, 499, 520, 610):
        c, t, want, blank = (canvases[x][k] if x != "list" else canvases["list"][k]
                             for x in ("list", "thresholds", "outputs", "blank"))
        if blank:
            with pytest.raises(sd.BlankDrawingError):
                sd.preprocess_pipeline(c, int(t))
        else:
            assert np.array_equal(sd.preprocess_pipeline(c, int(t)), want)
    with pytest.raises(sd.BlankDrawingError):
        sd.preprocess_pipeline(np.zeros((40, 30), dtype=np.uint8))
    with pytest.raises(ValueError):
        sd.preprocess_pipeline(np.zeros((3,), dtype=np.uint8))
    with pytest.raises(ValueError):
        sd.preprocess_pipeline(np.full((20, 20), 255, dtype=np.uint8), threshold=300)
    # the largest canvas the service accepts, one ink pixel in a corner
    big = np.zeros((1024, 1024), dtype=np.uint8)
    big[1023, 0] = 255
    from oracle import preprocess_oracle as P
    assert np.array_equal(sd.preprocess_pipeline(big), P.preprocess(big))


def test_host_normalisation_keeps_the_reference_mask():
    """preprocess._prepare (non-uint8 canvases, fractional thresholds, canvases
    over 1024 px): the uint8 canvas and integer threshold it hands the kernel
    give the reference's outputs (checked with the oracle's pipeline on CPU
    against oracle/gen_canvases_extra.py's reference fixtures)."""
    import os
    from oracle import preprocess_oracle as P
    from paper_1711_03637_b200.preprocess import MAX_SIDE, _prepare
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "canvases_extra.npz"))
    for k in range(6):
        cv, thr = z[f"canvas{k}"], float(z[f"threshold{k}"])
        thr = int(thr) if thr.is_integer() else thr
        arr, t = _prepare(cv, thr)
        assert arr.dtype == np.uint8 and isinstance(t, int) and 0 <= t <= 255
        assert max(arr.shape) <= MAX_SIDE
        assert np.array_equal(P.preprocess(arr, t), z[f"out{k}"]), k
    with pytest.raises(ValueError, match="threshold"):
        _prepare(np.zeros((4, 4), np.uint8), 256)
    with pytest.raises(ValueError, match="2-D"):
        _prepare(np.zeros(4, np.uint8), 128)
    blank, t = _prepare(np.zeros((1500, 20), np.uint8), 128)
    assert blank.shape == (1, 1) and not (blank >= t).any()
