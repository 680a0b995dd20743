"""Configuration types, constants and validation of the reference API.

Same names, fields, defaults and error behaviour as the reference package
``spikedigits`` (paths relative to /root/reference/pkg/src/spikedigits), so a
caller can switch imports without touching its code:

  LifParams / min_spiking_current      neurons.py:23-60
  EncodingParams / NetworkConfig       network.py:54-150
  single_synapse_rate_weight           network.py:80-101
  SpikeRecord / desired_spike_train    network.py:153-193
  FilterBank / default_filter_bank     filters.py:34-88
  LearnConfig / NumericFailureError    normad.py:36-52
  EpochStats                           normad.py:165-176
  as_pixel_image / as_pixel_batch / check_weights   validation.py:10-56

The wrappers in ``api.py`` also accept the reference's own objects (they only
read attributes), which is what ``shim.install()`` relies on.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

IMAGE_SIDE = 28
FEATURE_SIDE = 26
N_FEATURE_MAPS = 12
N_INPUTS = IMAGE_SIDE * IMAGE_SIDE
N_HIDDEN = N_FEATURE_MAPS * FEATURE_SIDE * FEATURE_SIDE
N_OUTPUTS = 10
N_FILTERS = N_FEATURE_MAPS

TAU_SYN_SLOW = 5e-3
TAU_SYN_FAST = 1.25e-3
TAU_LEARN = 1e-3
DEFAULT_LEARNING_RATE = 2e-7
DEFAULT_FILTER_DRIVE = 15e-9


# --------------------------------------------------------------------- neurons

@dataclass(frozen=True)
class LifParams:
    """LIF population constants in SI units (C, g_L, E_L, V_T, t_ref)."""

    capacitance: float = 300e-12
    leak_conductance: float = 30e-9
    rest_potential: float = -70e-3
    threshold: float = 20e-3
    refractory: float = 3e-3

    def __post_init__(self):
        checks = (
            (self.capacitance > 0, "capacitance must be positive"),
            (self.leak_conductance > 0, "leak_conductance must be positive"),
            (self.threshold > self.rest_potential, "threshold must exceed rest_potential"),
            (self.refractory >= 0, "refractory must be non-negative"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def tau_m(self) -> float:
        return self.capacitance / self.leak_conductance


def min_spiking_current(params: LifParams) -> float:
    """Rheobase g_L * (V_T - E_L)."""
    return params.leak_conductance * (params.threshold - params.rest_potential)


# --------------------------------------------------------------------- network

@dataclass(frozen=True)
class EncodingParams:
    """Pixel level k -> constant current i_0 + k * i_p."""

    i_0: float = 2700e-12
    i_p: float = 101.2e-12

    def __post_init__(self):
        if not self.i_0 > 0:
            raise ValueError("i_0 must be positive")
        if not self.i_p > 0:
            raise ValueError("i_p must be positive")


def single_synapse_rate_weight(params: LifParams, rate: float,
                               tau_slow: float = TAU_SYN_SLOW, tau_fast: float = TAU_SYN_FAST) -> float:
    """Weight at which one synapse carrying a `rate` train sustains that rate
    (mean-current approximation)."""
    if rate <= 0:
        raise ValueError("rate must be positive")
    recharge = 1.0 / rate - params.refractory
    if recharge <= 0:
        raise ValueError("rate is infeasible under the refractory period")
    needed = min_spiking_current(params) / -math.expm1(-recharge / params.tau_m)
    return needed / (rate * (tau_slow - tau_fast))


@dataclass(frozen=True)
class NetworkConfig:
    """Presentation timing, encoding and the three LIF populations."""

    t: float = 0.100
    dt: float = 1e-3
    desired_rate: float = 285.0
    inhibition_weight: Optional[float] = None
    encoding: EncodingParams = EncodingParams()
    input_lif: LifParams = LifParams()
    hidden_lif: LifParams = LifParams()
    output_lif: LifParams = LifParams()

    def __post_init__(self):
        if not (self.t > 0 and self.dt > 0):
            raise ValueError("t and dt must be positive")
        ratio = self.t / self.dt
        if abs(ratio - round(ratio)) > 1e-6 * max(1.0, ratio):
            raise ValueError(f"t/dt = {ratio} is not an integer number of steps")
        if self.desired_rate < 0:
            raise ValueError("desired_rate must be non-negative")
        if self.desired_rate * self.output_lif.refractory >= 1.0:
            raise ValueError("desired_rate is infeasible under the output refractory period")
        if not math.isclose(self.encoding.i_0, min_spiking_current(self.input_lif), rel_tol=1e-9):
            raise ValueError("encoding i_0 must equal the input layer rheobase")
        if self.inhibition_weight is None:
            inh = (-single_synapse_rate_weight(self.output_lif, self.desired_rate)
                   if self.desired_rate > 0 else 0.0)
            object.__setattr__(self, "inhibition_weight", inh)
        elif self.inhibition_weight > 0:
            raise ValueError("inhibition_weight must be non-positive")

    @property
    def n_steps(self) -> int:
        return int(round(self.t / self.dt))


@dataclass
class SpikeRecord:
    """Spike rasters of one presentation as per-neuron step-index lists."""

    input_spikes: list
    hidden_spikes: list
    output_spikes: list
    output_counts: np.ndarray

    def __post_init__(self):
        counts = np.asarray(self.output_counts, dtype=np.int64)
        if counts.shape != (N_OUTPUTS,):
            raise ValueError("output_counts must have 10 entries")
        if [len(s) for s in self.output_spikes] != counts.tolist():
            raise ValueError("output counts disagree with spike lists")
        self.output_counts = counts


def desired_spike_train(t: float, dt: float, rate: float, refractory: float = 3e-3) -> np.ndarray:
    """Target spike steps: period = round(1/(rate*dt)), first spike one period in."""
    if not (t > 0 and dt > 0):
        raise ValueError("t and dt must be positive")
    if rate < 0:
        raise ValueError("rate must be non-negative")
    if rate == 0:
        return np.empty(0, dtype=np.int64)
    if rate * refractory >= 1.0:
        raise ValueError(f"rate {rate} Hz infeasible: period shorter than refractory {refractory}")
    return np.arange(desired_period(t, dt, rate) - 1, int(round(t / dt)),
                     desired_period(t, dt, rate), dtype=np.int64)


def desired_period(t: float, dt: float, rate: float) -> int:
    """Steps between target spikes (0 when the target train is empty)."""
    if rate == 0:
        return 0
    return max(1, int(math.floor(1.0 / (rate * dt) + 0.5)))


def parameter_count() -> int:
    return N_HIDDEN * N_OUTPUTS


def zero_weights() -> np.ndarray:
    return np.zeros((N_HIDDEN, N_OUTPUTS), dtype=np.float64)


def classify(record) -> int:
    """argmax of the output counts; ties go to the lowest digit."""
    counts = np.asarray(getattr(record, "output_counts", record))
    if counts.shape != (N_OUTPUTS,):
        raise ValueError("expected 10 output counts")
    return int(np.argmax(counts))


# --------------------------------------------------------------------- filters

_EDGE = (
    ((1, 2, 1), (0, 0, 0), (-1, -2, -1)),
    ((1, 0, -1), (2, 0, -2), (1, 0, -1)),
    ((2, 1, 0), (1, 0, -1), (0, -1, -2)),
    ((0, 1, 2), (-1, 0, 1), (-2, -1, 0)),
)


def _corner(r0: int, c0: int) -> np.ndarray:
    k = np.full((3, 3), -4.0)
    k[r0:r0 + 2, c0:c0 + 2] = 5.0
    return k


@dataclass(frozen=True)
class FilterBank:
    """Twelve 3x3 kernels plus per-filter current gains (immutable)."""

    kernels: np.ndarray
    gains: np.ndarray

    def __post_init__(self):
        k = np.array(self.kernels, dtype=np.float64, copy=True)
        g = np.array(self.gains, dtype=np.float64, copy=True)
        if k.shape != (N_FILTERS, 3, 3):
            raise ValueError(f"expected {(N_FILTERS, 3, 3)} kernels, got {k.shape}")
        if g.shape != (N_FILTERS,):
            raise ValueError(f"expected {N_FILTERS} gains, got {g.shape}")
        if not (np.all(np.isfinite(k)) and np.all(np.isfinite(g))):
            raise ValueError("filter bank contains non-finite values")
        k.setflags(write=False)
        g.setflags(write=False)
        object.__setattr__(self, "kernels", k)
        object.__setattr__(self, "gains", g)

    @property
    def weighted(self) -> np.ndarray:
        return self.kernels * self.gains[:, None, None]


def default_filter_bank(drive: float = DEFAULT_FILTER_DRIVE) -> FilterBank:
    """4 Sobel-style edges, their negations, 4 corner contrasts; each gain is
    drive / (sum of the kernel's positive cells)."""
    edges = np.array(_EDGE)          # negate as integers: zero taps stay +0.0 as in filters.py:76-79
    kernels = np.concatenate([edges, -edges]).astype(np.float64)
    kernels = np.concatenate([kernels, np.stack([_corner(0, 0), _corner(0, 1), _corner(1, 0), _corner(1, 1)])])
    return FilterBank(kernels=kernels, gains=drive / np.clip(kernels, 0.0, None).sum(axis=(1, 2)))


# --------------------------------------------------------------------- learning

class NumericFailureError(RuntimeError):
    """Training produced non-finite weights."""


@dataclass
class LearnConfig:
    learning_rate: float = DEFAULT_LEARNING_RATE
    norm_epsilon: float = 1e-12

    def __post_init__(self):
        if not self.learning_rate > 0:
            raise ValueError("learning_rate must be positive")
        if self.norm_epsilon < 0:
            raise ValueError("norm_epsilon must be non-negative")


@dataclass
class EpochStats:
    n_images: int = 0
    n_errors: int = 0
    wall_seconds: float = 0.0
    error_counts: list = field(default_factory=lambda: [0] * N_OUTPUTS)

    @property
    def error_rate(self) -> float:
        return self.n_errors / self.n_images if self.n_images else 0.0


# --------------------------------------------------------------------- validation

def as_pixel_image(x) -> np.ndarray:
    """(28,28) or (784,) whole-number levels 0..255 -> (28,28) uint8."""
    arr = np.asarray(x)
    if arr.shape == (N_INPUTS,):
        arr = arr.reshape(IMAGE_SIDE, IMAGE_SIDE)
    if arr.shape != (IMAGE_SIDE, IMAGE_SIDE):
        raise ValueError(f"expected a 28x28 image, got shape {arr.shape}")
    if arr.dtype == np.uint8:
        return arr
    vals = arr.astype(np.float64)
    if not np.all(np.isfinite(vals)):
        raise ValueError("image contains non-finite values")
    if np.any((vals < 0) | (vals > 255)):
        raise ValueError("pixel levels must lie in 0..255")
    if np.any(vals != np.round(vals)):
        raise ValueError("pixel levels must be whole numbers")
    return vals.astype(np.uint8)


def as_pixel_batch(X) -> np.ndarray:
    """(n,784) or (n,28,28) -> (n,28,28) uint8 (per-image checks as above)."""
    arr = np.asarray(X)
    if arr.ndim == 1:
        raise ValueError("expected a batch of images, got a single vector")
    if arr.ndim == 2 and arr.shape[1] == N_INPUTS:
        arr = arr.reshape(-1, IMAGE_SIDE, IMAGE_SIDE)
    if arr.ndim != 3 or arr.shape[1:] != (IMAGE_SIDE, IMAGE_SIDE):
        raise ValueError(f"expected (n, 784) or (n, 28, 28), got shape {arr.shape}")
    if arr.dtype == np.uint8:
        return arr
    return np.stack([as_pixel_image(im) for im in arr])


def check_weights(w, shape=None) -> np.ndarray:
    """2-D finite float64 weights (optionally of an exact shape)."""
    arr = np.asarray(w, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"weights must be 2-D, got shape {arr.shape}")
    if shape is not None and arr.shape != tuple(shape):
        raise ValueError(f"expected weights of shape {tuple(shape)}, got {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError("weights contain non-finite values")
    return arr
