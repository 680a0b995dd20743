"""ctypes binding of the C ABI in include/snn_b200.h (libsnn_b200.so, in-tree).

The shared library is the product: there is no CPU fallback.  Loading fails
loudly when the library is missing (run ``python -c "import __graft_entry__ as
g; g.build()"`` or ``python -m paper_1711_03637_b200.build``).
"""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsnn_b200.so")


ABI_VERSION = 2   # SNN_ABI_VERSION of include/snn_b200.h

SNN_OK = 0
SNN_ENOMEM = 12
SNN_EINVAL = 22
SNN_ENONFINITE = 1001
SNN_ECUDA = 1002

MAX_TILES = 22
TILE = 32
NORMAD_DEFAULT = 4   # snn_set_normad_cluster default: the speculative-scan kernel
RASTER_CHUNK = 8


def raster_bytes(n_images: int, n_steps: int) -> int:
    """Upper bound of the compact hidden raster of n images (include/snn_b200.h)."""
    return n_images * MAX_TILES * (-(-n_steps // RASTER_CHUNK)) * 2 * TILE * RASTER_CHUNK

_d = ctypes.c_double
_vp = ctypes.c_void_p


class LifC(ctypes.Structure):
    _fields_ = [("g", _d), ("el", _d), ("vt", _d), ("beta", _d), ("refr", _d)]


class ConstsC(ctypes.Structure):
    _fields_ = [
        ("n_steps", ctypes.c_int32),
        ("desired_period", ctypes.c_int32),
        ("dt", _d),
        ("i0", _d),
        ("ip", _d),
        ("lif_in", LifC),
        ("lif_hid", LifC),
        ("lif_out", LifC),
        ("decay_slow", _d),
        ("decay_fast", _d),
        ("decay_learn", _d),
        ("dhat_scale", _d),
        ("inhibition", _d),
        ("learning_rate", _d),
        ("norm_eps", _d),
        ("taps", (_d * 9) * 12),
    ]


class InferOutC(ctypes.Structure):
    _fields_ = [(name, _vp) for name in
                ("counts", "raster", "tile_pos", "n_tiles", "tile_base", "out_raster", "ff", "v_out", "v_hid",
                 "near_ties", "hidden_redo")]


# (name, restype, argtypes) -- one row per declaration in include/snn_b200.h
SIGNATURES = [
    ("snn_abi_version", ctypes.c_int, []),
    ("snn_last_error", ctypes.c_char_p, []),
    ("snn_input_table", ctypes.c_int, [ctypes.POINTER(ConstsC), _vp, _vp, _vp]),
    ("snn_infer_workspace", ctypes.c_size_t, [ctypes.POINTER(ConstsC), ctypes.c_int64]),
    ("snn_infer", ctypes.c_int, [ctypes.POINTER(ConstsC), _vp, ctypes.c_int64, _vp, _vp,
                                 ctypes.POINTER(InferOutC), _vp, ctypes.c_size_t, _vp]),
    ("snn_profile_events", None, [_vp, _vp]),
    ("snn_profile_stage_events", None, [_vp, ctypes.c_int]),
    ("snn_set_pipeline", None, [ctypes.c_int64, ctypes.c_int]),
    ("snn_set_normad_cluster", None, [ctypes.c_int]),
    ("snn_set_output_dist", None, [ctypes.c_int]),
    ("snn_set_hidden_resident", None, [ctypes.c_int]),
    ("snn_normad_phase_clocks", None, [_vp]),
    ("snn_normad_skip", None, [ctypes.c_int]),
    ("snn_train_chunk", ctypes.c_int64, [ctypes.POINTER(ConstsC), ctypes.c_int64]),
    ("snn_train_workspace", ctypes.c_size_t, [ctypes.POINTER(ConstsC), ctypes.c_int64]),
    ("snn_preprocess", ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp]),
    ("snn_train", ctypes.c_int, [ctypes.POINTER(ConstsC), _vp, _vp, ctypes.c_int64, _vp, _vp, _vp,
                                 _vp, _vp, ctypes.c_size_t, _vp]),
]

_LIB = None


def load():
    """Load (once) and type the in-tree shared library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    # profiling scripts only: an alternative in-tree build (build.py --profile)
    path = os.environ.get("SNN_B200_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: the CUDA extension has not been built "
            "(python -m paper_1711_03637_b200.build). There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.snn_abi_version() != ABI_VERSION:
        raise ImportError("libsnn_b200.so ABI version mismatch")
    _LIB = lib
    return lib


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"snn native error {code}: {msg}")
        self.code = code


def check(rc: int):
    if rc != SNN_OK:
        msg = load().snn_last_error().decode(errors="replace")
        if rc == SNN_EINVAL:
            raise ValueError(msg)
        raise NativeError(rc, msg)
