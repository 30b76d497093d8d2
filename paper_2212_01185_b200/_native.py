"""ctypes binding of liblpic_b200.so (include/lpic_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import LpicError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LPIC_LIB", os.path.join(_HERE, "liblpic_b200.so"))   # (override: A/B builds)

LPIC_OK = 0
LPIC_E_ARG = -1
LPIC_E_CUDA = -2
LPIC_E_UNSUPPORTED = -3
LPIC_E_NOMEM = -4
LPIC_S_NONFINITE = 1
LPIC_S_CORRUPT = 2
LPIC_S_CAPACITY = 4
LPIC_S_INTERNAL = 8
PREC_COMPAT = 0
PREC_FAST = 1

# every symbol include/lpic_b200.h declares
EXPORTS = (
    "lpic_version", "lpic_last_error", "lpic_model_create", "lpic_model_destroy",
    "lpic_model_set_precision", "lpic_model_fingerprint", "lpic_fnv1a64", "lpic_forward_taps",
    "lpic_forward_full", "lpic_channel_cdfs", "lpic_rc_encode_streams", "lpic_rc_decode_tables",
    "lpic_encode_batch_device", "lpic_decode_batch_device", "lpic_encode_batch", "lpic_decode_batch",
    "lpic_last_launch_count", "lpic_true_symbol_probs", "lpic_theoretical_bits", "lpic_network_coding_order",
    "lpic_mixture_loss_grad", "lpic_quantized_cdf", "lpic_rc_dec_create", "lpic_rc_dec_decode",
    "lpic_rc_dec_destroy", "lpic_mixture_loss_grad_f64",
)


class NativeUnavailable(LpicError):
    """liblpic_b200.so could not be loaded or no CUDA device is present."""


_lib = None

_vp = C.c_void_p
_i64 = C.c_int64
_i = C.c_int


def load(path: str = LIB_PATH):
    """Load the shared library and declare signatures (no CUDA calls)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing; build it with `python -m paper_2212_01185_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(path)
    L.lpic_version.restype = _i
    L.lpic_last_error.restype = C.c_char_p
    L.lpic_model_create.argtypes = [_vp] * 6 + [_i] * 5 + [C.POINTER(_vp)]
    L.lpic_model_destroy.argtypes = [_vp]
    L.lpic_model_set_precision.argtypes = [_vp, _i]
    L.lpic_model_fingerprint.argtypes = [_vp]
    L.lpic_model_fingerprint.restype = C.c_uint64
    L.lpic_fnv1a64.argtypes = [_vp, _i64]
    L.lpic_fnv1a64.restype = C.c_uint64
    L.lpic_forward_taps.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.lpic_forward_full.argtypes = [_vp, _vp, _i, _i, _vp, _vp]
    L.lpic_channel_cdfs.argtypes = [_vp, _i64, _i, _i, _i, _i, _vp, _vp, _vp, _vp]
    L.lpic_rc_encode_streams.argtypes = [_vp, _vp, _vp, _i, _vp, _i64, _vp, _vp, _vp]
    L.lpic_rc_decode_tables.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp, _vp]
    L.lpic_encode_batch_device.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.lpic_decode_batch_device.argtypes = [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]
    L.lpic_encode_batch.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp, _i64, _vp, _vp, _vp, _vp]
    L.lpic_decode_batch.argtypes = [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp]
    L.lpic_last_launch_count.argtypes = [_vp]
    L.lpic_true_symbol_probs.argtypes = [_vp, _i64, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]
    L.lpic_theoretical_bits.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp, _vp]
    L.lpic_network_coding_order.argtypes = [_vp, _vp, _i, _i, _i, _i, _vp, _vp]
    L.lpic_mixture_loss_grad.argtypes = [_vp, _vp, _i64, _i, _i, _vp, _vp, _vp]
    L.lpic_mixture_loss_grad_f64.argtypes = [_vp, _vp, _i64, _i, _i, _vp, _vp, _vp]
    L.lpic_quantized_cdf.argtypes = [_vp, _vp, _vp, _i64, _i, _i, _vp, _vp, _vp, _vp]
    L.lpic_rc_dec_create.argtypes = [_vp, _i64, C.POINTER(_vp)]
    L.lpic_rc_dec_decode.argtypes = [_vp, _vp, _vp]
    L.lpic_rc_dec_destroy.argtypes = [_vp]
    _lib = L
    return L


def require_cuda():
    """The product path needs a CUDA device; fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the LPIC B200 path has no CPU fallback")
    return load()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.lpic_last_error().decode(errors="replace") if _lib is not None else ""
        if rc == LPIC_E_UNSUPPORTED:
            raise LpicError(f"{what}: unsupported on the GPU path: {msg}")
        if rc == LPIC_E_ARG:
            raise ValueError(f"{what}: {msg}")
        raise LpicError(f"{what} failed ({rc}): {msg}")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
