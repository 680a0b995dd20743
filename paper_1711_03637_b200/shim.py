"""Reroute an importable reference package (``spikedigits``) onto the GPU.

The reference binds its hot-path functions with ``from .x import y``, so each
importing module holds its own reference; ``install()`` rebinds every one of
them and makes the GPU wrappers raise and return the
reference's own exception / record / stats classes.  ``uninstall()`` restores.

``install(count=True)`` also counts the calls that reach each GPU entry point
(``call_counts()``), so a harness can show that the reference's own code paths
really ran on the GPU.  ``install(warm=True)`` (the default) also wraps the
service's ``create_app`` so that the CUDA context, the library, the device
weights, the input table and the batch-1 CUDA graph of the service's default
configuration are built when the app is created, not on the first request
(PAPER.md:160 moves the ~300 ms CUDA initialisation to startup).

Command line: ``python -m paper_1711_03637_b200.shim -m spikedigits.cli train
...`` runs any module of the reference (here its CLI) with the shim installed.
"""
from __future__ import annotations

import functools
import importlib
import runpy
import sys
import threading

from . import api, preprocess

# (module, attribute, replacement)
_BINDINGS = [
    ("spikedigits.network", "run_presentation", api.run_presentation),
    ("spikedigits.network", "forward_pass", api.forward_pass),
    ("spikedigits.evaluate", "run_presentation", api.run_presentation),
    ("spikedigits.evaluate", "batch_counts", api.batch_counts),
    ("spikedigits.normad", "run_presentation", api.run_presentation),
    ("spikedigits.normad", "train_presentation", api.train_presentation),
    ("spikedigits.normad", "train_epoch", api.train_epoch),
    ("spikedigits.cli", "run_presentation", api.run_presentation),
    ("spikedigits.cli", "train_epoch", api.train_epoch),
    ("spikedigits.service", "run_presentation", api.run_presentation),
    ("spikedigits.estimator", "batch_counts", api.batch_counts),
    ("spikedigits.estimator", "train_epoch", api.train_epoch),
    ("spikedigits", "forward_pass", api.forward_pass),
    ("spikedigits", "train_epoch", api.train_epoch),
    ("spikedigits.cli", "preprocess_pipeline", preprocess.preprocess_pipeline),
    ("spikedigits.service", "preprocess_pipeline", preprocess.preprocess_pipeline),
    ("spikedigits.strokes", "preprocess_pipeline", preprocess.preprocess_pipeline),
    ("spikedigits.preprocess", "preprocess_pipeline", preprocess.preprocess_pipeline),
]

_saved: list = []
_counts: dict = {}
_counts_lock = threading.Lock()


def _counting(name: str, fn):
    @functools.wraps(fn)
    def wrapper(*a, **k):
        with _counts_lock:
            _counts[name] = _counts.get(name, 0) + 1
        return fn(*a, **k)
    return wrapper


def call_counts() -> dict:
    """Calls per GPU entry point since install(count=True)."""
    with _counts_lock:
        return dict(_counts)


def warm_service(app) -> float:
    """Build everything the service's first request would otherwise build:
    CUDA context, library, device weights, input table and the batch-1 CUDA
    graph of the app's default (t_ms, dt_ms).  Returns the seconds it took;
    no-op (0.0) for an app without a checkpoint."""
    import dataclasses
    import time

    import numpy as np

    eng_ref = getattr(getattr(app, "state", None), "engine", None)
    loaded = getattr(eng_ref, "_loaded", None)
    if loaded is None:
        return 0.0
    t0 = time.perf_counter()
    cfg = dataclasses.replace(loaded.cfg, t=eng_ref.t_ms * 1e-3, dt=eng_ref.dt_ms * 1e-3)
    api.run_presentation(np.zeros((28, 28), dtype=np.uint8), loaded.weights, loaded.filters, cfg)
    return time.perf_counter() - t0


def _warming_create_app(create_app):
    @functools.wraps(create_app)
    def wrapper(*a, **k):
        app = create_app(*a, **k)
        app.state.gpu_warmup_s = warm_service(app)
        return app
    return wrapper


def install(count: bool = False, warm: bool = True) -> int:
    """Rebind the reference's hot-path names; returns how many were bound."""
    if _saved:
        return len(_saved)
    normad = importlib.import_module("spikedigits.normad")
    network = importlib.import_module("spikedigits.network")
    api._NUMERIC_ERROR = normad.NumericFailureError
    api._EPOCH_STATS = normad.EpochStats
    api._SPIKE_RECORD = network.SpikeRecord
    preprocess._BLANK_ERROR = importlib.import_module("spikedigits.preprocess").BlankDrawingError
    for mod_name, attr, fn in _BINDINGS:
        try:
            mod = importlib.import_module(mod_name)
        except ImportError:  # optional entry points (fastapi / sklearn missing)
            continue
        if hasattr(mod, attr):
            _saved.append((mod, attr, getattr(mod, attr)))
            setattr(mod, attr, _counting(fn.__name__, fn) if count else fn)
    if warm:
        try:
            service = importlib.import_module("spikedigits.service")
        except ImportError:
            service = None
        if service is not None and hasattr(service, "create_app"):
            _saved.append((service, "create_app", service.create_app))
            service.create_app = _warming_create_app(service.create_app)
    return len(_saved)


def uninstall() -> None:
    from .params import EpochStats, NumericFailureError, SpikeRecord
    while _saved:
        mod, attr, old = _saved.pop()
        setattr(mod, attr, old)
    api._NUMERIC_ERROR = NumericFailureError
    api._EPOCH_STATS = EpochStats
    api._SPIKE_RECORD = SpikeRecord
    preprocess._BLANK_ERROR = preprocess.BlankDrawingError


def main(argv=None) -> None:
    """``python -m paper_1711_03637_b200.shim -m MODULE [ARGS...]``: run a
    module of the reference (e.g. its CLI) with the GPU path installed."""
    argv = list(sys.argv[1:] if argv is None else argv)
    if len(argv) < 2 or argv[0] != "-m":
        raise SystemExit("usage: python -m paper_1711_03637_b200.shim -m MODULE [ARGS...]")
    install()
    mod = argv[1]
    sys.argv = [mod] + argv[2:]
    runpy.run_module(mod, run_name="__main__", alter_sys=True)


if __name__ == "__main__":
    main()
