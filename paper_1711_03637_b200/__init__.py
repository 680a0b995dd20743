"""B200-native spiking-digit hot path: SNN inference and NormAD training.

A from-scratch sm_100a implementation of the hot path of the reference
package ``spikedigits`` (arXiv 1711.03637), behind the reference's own Python
API.  ``import paper_1711_03637_b200 as sd`` and use it like ``spikedigits``;
or call ``paper_1711_03637_b200.shim.install()`` to reroute an installed
``spikedigits`` (its CLI, HTTP service and sklearn estimator) onto the GPU.
"""
from .api import (EvalReport, batch_counts, batch_counts_device, evaluate_dataset, forward_pass,
                  run_presentation, train_epoch, train_presentation)
from .preprocess import BlankDrawingError, preprocess_batch, preprocess_pipeline
from .params import (DEFAULT_FILTER_DRIVE, DEFAULT_LEARNING_RATE, N_HIDDEN, N_INPUTS, N_OUTPUTS,
                     EncodingParams, EpochStats, FilterBank, LearnConfig, LifParams, NetworkConfig,
                     NumericFailureError, SpikeRecord, as_pixel_batch, as_pixel_image, check_weights,
                     classify, default_filter_bank, desired_spike_train, min_spiking_current,
                     parameter_count, single_synapse_rate_weight, zero_weights)

__version__ = "0.1.0"

__all__ = [
    "run_presentation", "forward_pass", "batch_counts", "batch_counts_device", "evaluate_dataset",
    "EvalReport", "train_presentation", "train_epoch", "EncodingParams", "EpochStats", "FilterBank",
    "LearnConfig", "LifParams", "NetworkConfig", "NumericFailureError", "SpikeRecord", "classify",
    "default_filter_bank", "desired_spike_train", "min_spiking_current", "parameter_count",
    "single_synapse_rate_weight", "zero_weights", "as_pixel_batch", "as_pixel_image", "check_weights",
    "N_HIDDEN", "N_INPUTS", "N_OUTPUTS", "DEFAULT_FILTER_DRIVE", "DEFAULT_LEARNING_RATE",
    "preprocess_pipeline", "preprocess_batch", "BlankDrawingError",
]
