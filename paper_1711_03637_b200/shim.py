"""Reroute an importable reference package (``spikedigits``) onto the GPU.

The reference binds its hot-path functions with ``from .x import y``, so each
importing module holds its own reference; ``install()`` rebinds every one of
them and makes the GPU wrappers raise and return the
reference's own exception / record / stats classes.  ``uninstall()`` restores.
"""
from __future__ import annotations

import importlib

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
]

_saved: list = []


def install() -> int:
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
            setattr(mod, attr, fn)
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
