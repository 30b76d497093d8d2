"""Model configuration, weights, LPWT files and the GPU forward entry points.

Drop-in mirror of /root/reference/pkg/src/lpic/network.py: the same names,
argument meaning and error behaviour.  The forward passes run on the B200
through liblpic_b200.so (k_forward_full / k_forward_taps, canonical float32
order, bit-identical to kernels.forward_full_f32, kernels.py:88-136); there
is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import struct
import threading
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _native
from .errors import LpicError

WEIGHT_MAGIC = b"LPWT"
WEIGHT_VERSION = 1
LEAKY_SLOPE = 0.01


class Distribution(IntEnum):
    GAUSSIAN = 0
    LOGISTIC = 1


@dataclass(frozen=True)
class ModelConfig:
    """K mixtures, C filters, L conv layers, kernel half-width h
    (network.py:33-74 of the reference)."""

    mixtures: int = 3
    filters: int = 128
    layers: int = 5
    kernel_half: int = 2
    distribution: Distribution = Distribution.GAUSSIAN

    def __post_init__(self):
        if self.mixtures < 1:
            raise ValueError("mixtures must be positive")
        if self.filters < 1:
            raise ValueError("filters must be positive")
        if self.layers < 3:
            raise ValueError("need at least masked + hidden + output layers")
        if self.kernel_half < 1:
            raise ValueError("kernel_half must be positive")
        if self.distribution not in (Distribution.GAUSSIAN, Distribution.LOGISTIC):
            raise ValueError("unknown distribution")

    @property
    def param_channels(self) -> int:
        return 12 * self.mixtures

    @property
    def hidden_count(self) -> int:
        return self.layers - 2

    @property
    def tap_count(self) -> int:
        h = self.kernel_half
        return (2 * h + 1) * h + h


REFERENCE_CONFIG = ModelConfig()


def causal_taps(kernel_half: int) -> np.ndarray:
    """(T, 2) tap offsets: the h rows above the centre (dj = -h..h), then
    the h pixels to its left (kernels.py:42-55)."""
    h = int(kernel_half)
    rows = [(di, dj) for di in range(-h, 0) for dj in range(-h, h + 1)]
    rows += [(0, dj) for dj in range(-h, 0)]
    return np.asarray(rows, dtype=np.int64)


@dataclass
class Weights:
    masked_w: np.ndarray  # (T, 3, C)
    masked_b: np.ndarray  # (C,)
    hidden_w: np.ndarray  # (L-2, C, C) out x in
    hidden_b: np.ndarray  # (L-2, C)
    out_w: np.ndarray     # (M, C)
    out_b: np.ndarray     # (M,)

    def tensors(self):
        return [self.masked_w, self.masked_b, self.hidden_w, self.hidden_b, self.out_w, self.out_b]

    def copy(self) -> "Weights":
        return Weights(*[t.copy() for t in self.tensors()])


def weight_shapes(cfg: ModelConfig):
    T, Cf, M, NH = cfg.tap_count, cfg.filters, cfg.param_channels, cfg.hidden_count
    return [("masked_w", (T, 3, Cf)), ("masked_b", (Cf,)), ("hidden_w", (NH, Cf, Cf)),
            ("hidden_b", (NH, Cf)), ("out_w", (M, Cf)), ("out_b", (M,))]


def zero_weights(cfg: ModelConfig) -> Weights:
    return Weights(*[np.zeros(s, np.float32) for _, s in weight_shapes(cfg)])


def _uniform_init(cfg: ModelConfig, rng: np.random.Generator, bound_of) -> Weights:
    # draw order masked_w, hidden_w, out_w; biases stay zero (network.py:120-134)
    w = zero_weights(cfg)
    T, Cf, M = cfg.tap_count, cfg.filters, cfg.param_channels
    for name, fan_in, fan_out in (("masked_w", 3 * T, Cf), ("hidden_w", Cf, Cf), ("out_w", Cf, M)):
        t = getattr(w, name)
        b = bound_of(fan_in, fan_out)
        t[:] = rng.uniform(-b, b, t.shape).astype(np.float32)
    return w


def glorot_weights(cfg: ModelConfig, rng: np.random.Generator) -> Weights:
    """Uniform(-b, b), b = sqrt(6 / (fan_in + fan_out)); zero biases."""
    return _uniform_init(cfg, rng, lambda fi, fo: float(np.sqrt(6.0 / (fi + fo))))


def kaiming_weights(cfg: ModelConfig, rng: np.random.Generator) -> Weights:
    """Harness 'Kaiming seed s' init: uniform with
    b = sqrt(2/(1+0.01^2)) * sqrt(3/fan_in), Glorot's draw order, zero biases.
    Not part of the reference (which only has Glorot)."""
    gain = float(np.sqrt(2.0 / (1.0 + 0.01 ** 2)))
    return _uniform_init(cfg, rng, lambda fi, fo: gain * float(np.sqrt(3.0 / fi)))


def count_parameters(cfg: ModelConfig) -> int:
    return int(sum(int(np.prod(s)) for _, s in weight_shapes(cfg)))


def estimate_macs(cfg: ModelConfig, height: int, width: int) -> int:
    c = cfg.filters
    per_px = cfg.tap_count * 3 * c + cfg.hidden_count * c * c + c * cfg.param_channels
    return per_px * height * width


def check_weights(w: Weights, cfg: ModelConfig) -> None:
    for (name, shape), t in zip(weight_shapes(cfg), w.tensors()):
        if t.shape != shape:
            raise LpicError(f"weight tensor {name} has shape {t.shape}, expected {shape}")
        if t.dtype != np.float32:
            raise LpicError(f"weight tensor {name} must be float32")


# ---------------------------------------------------------------------------
# normalisation (network.py:172-183): float32 x / 127.5 - 1 with true division
# ---------------------------------------------------------------------------
_NORM_LUT = (np.arange(256, dtype=np.float32) / np.float32(127.5) - np.float32(1.0)).astype(np.float32)


def normalize(image: np.ndarray) -> np.ndarray:
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValueError("expected an HxWx3 image")
    return image.astype(np.float32) / np.float32(127.5) - np.float32(1.0)


def normalize_value(v: int) -> np.float32:
    return np.float32(_NORM_LUT[int(v)])


def leaky_relu(x: float) -> float:
    return x if x >= 0 else LEAKY_SLOPE * x


# ---------------------------------------------------------------------------
# LPWT weight file + FNV-1a fingerprint (network.py:255-322), hashed natively
# ---------------------------------------------------------------------------
def fnv1a64(data: bytes) -> int:
    L = _native.load()
    buf = C.create_string_buffer(bytes(data), len(data)) if len(data) else C.create_string_buffer(1)
    return int(L.lpic_fnv1a64(buf, len(data)))


def serialize_weights(w: Weights, cfg: ModelConfig) -> bytes:
    check_weights(w, cfg)
    if max(cfg.filters, cfg.mixtures, cfg.layers, cfg.kernel_half) > 255:
        raise LpicError("config fields must fit in one byte each")
    head = WEIGHT_MAGIC + struct.pack("<BBBBBB", WEIGHT_VERSION, cfg.mixtures, cfg.filters,
                                      cfg.layers, cfg.kernel_half, int(cfg.distribution))
    return head + b"".join(np.ascontiguousarray(t, dtype="<f4").tobytes() for t in w.tensors())


def weight_fingerprint(w: Weights, cfg: ModelConfig) -> int:
    return fnv1a64(serialize_weights(w, cfg))


def save_weights(path, w: Weights, cfg: ModelConfig) -> int:
    payload = serialize_weights(w, cfg)
    fp = fnv1a64(payload)
    with open(path, "wb") as f:
        f.write(payload + struct.pack("<Q", fp))
    return fp


def load_weights(path) -> tuple[Weights, ModelConfig]:
    with open(path, "rb") as f:
        blob = f.read()
    if len(blob) < 18 or blob[:4] != WEIGHT_MAGIC:
        raise LpicError(f"{path}: not a weight file")
    body, (fp,) = blob[:-8], struct.unpack("<Q", blob[-8:])
    if fnv1a64(body) != fp:
        raise LpicError(f"{path}: fingerprint mismatch, file is corrupt")
    version, K, Cf, L, h, dist = struct.unpack("<BBBBBB", body[4:10])
    if version != WEIGHT_VERSION:
        raise LpicError(f"{path}: unsupported weight format version {version}")
    cfg = ModelConfig(mixtures=K, filters=Cf, layers=L, kernel_half=h, distribution=Distribution(dist))
    w = zero_weights(cfg)
    pos = 10
    for t in w.tensors():
        nbytes = t.size * 4
        if pos + nbytes > len(body):
            raise LpicError(f"{path}: truncated weight file")
        t[:] = np.frombuffer(body, dtype="<f4", count=t.size, offset=pos).reshape(t.shape)
        pos += nbytes
    if pos != len(body):
        raise LpicError(f"{path}: trailing bytes in weight file")
    return w, cfg


# ---------------------------------------------------------------------------
# GPU model handles (weights uploaded once per content fingerprint and device)
# ---------------------------------------------------------------------------
class GpuModel:
    """Owns an lpic_model_t: padded device weights + cached workspace."""

    def __init__(self, w: Weights, cfg: ModelConfig, precision: int = _native.PREC_COMPAT):
        L = _native.require_cuda()
        check_weights(w, cfg)
        self.cfg = cfg
        self._keep = [np.ascontiguousarray(t, dtype=np.float32) for t in w.tensors()]
        h = C.c_void_p()
        _native.check(L.lpic_model_create(*[t.ctypes.data for t in self._keep], cfg.mixtures, cfg.filters,
                                          cfg.layers, cfg.kernel_half, int(cfg.distribution), C.byref(h)),
                      "lpic_model_create")
        self.handle = h.value
        self.fingerprint = int(L.lpic_model_fingerprint(self.handle))
        if precision != _native.PREC_COMPAT:
            _native.check(L.lpic_model_set_precision(self.handle, precision), "lpic_model_set_precision")
        self.lock = threading.Lock()

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _native._lib is not None:
                _native._lib.lpic_model_destroy(self.handle)
        except Exception:
            pass


_MODELS: "OrderedDict" = None          # LRU of device handles (see gpu_model)
MODEL_CACHE_SIZE = 4
_PRECISION = {"compat": _native.PREC_COMPAT, "fast": _native.PREC_FAST}
_precision = "compat"
# FAST containers carry the weight fingerprint XOR this tag ("FAST" fp16x3),
# so a FAST stream presented to a compat decoder -- this library in compat
# precision or the CPU reference -- fails the fingerprint gate
# (FingerprintMismatchError, codec.py:197-199 of the reference) instead of
# silently decoding a wrong image, and vice versa.
FAST_FINGERPRINT_TAG = 0x4641535466703136


def set_precision(name: str) -> None:
    """Select the network arithmetic of every subsequent encode/decode.

    "compat" (default): the reference's canonical float32 order -- raw
    parameters bit-identical to the CPU reference, streams interchangeable
    with it.  "fast": tcgen05 tensor-core GEMMs with the fp16x3 split (raw
    within ~1e-5 relative); such streams round-trip on this library only and
    must be decoded with precision "fast" too.  FAST containers are tagged
    (``container_fingerprint``) so any other decoder refuses them.
    """
    global _precision
    if name not in _PRECISION:
        raise ValueError(f"precision must be one of {sorted(_PRECISION)}")
    _precision = name


def get_precision() -> str:
    return _precision


def container_fingerprint(w: Weights, cfg: ModelConfig, precision: str | None = None) -> int:
    """The fingerprint written into (and required from) a container: the
    weight fingerprint (network.py:264-281 of the reference) in compat
    precision, tagged in FAST precision."""
    fp = weight_fingerprint(w, cfg)
    if (precision or _precision) == "fast":
        fp ^= FAST_FINGERPRINT_TAG
    return fp


def gpu_model(w: Weights, cfg: ModelConfig) -> GpuModel:
    """The device handle for (weights, config, device, precision), from a
    small LRU: evicted handles free their device weights and workspaces."""
    global _MODELS
    import torch
    from collections import OrderedDict
    _native.require_cuda()
    if _MODELS is None:
        _MODELS = OrderedDict()
    key = (weight_fingerprint(w, cfg), cfg, torch.cuda.current_device(), _precision)
    m = _MODELS.get(key)
    if m is None:
        m = GpuModel(w, cfg, _PRECISION[_precision])
        _MODELS[key] = m
        while len(_MODELS) > MODEL_CACHE_SIZE:
            _MODELS.popitem(last=False)
    else:
        _MODELS.move_to_end(key)
    return m


def release_models() -> None:
    """Drop every cached device handle (frees their device memory once no
    caller holds them)."""
    if _MODELS is not None:
        _MODELS.clear()


def _kernel_call_taps(tap_values: np.ndarray, w: Weights, cfg: ModelConfig) -> np.ndarray:
    import torch
    m = gpu_model(w, cfg)
    N = tap_values.shape[0]
    out = np.empty((N, cfg.param_channels), np.float32)
    if N == 0:
        return out
    d_taps = torch.from_numpy(np.ascontiguousarray(tap_values, dtype=np.float32)).cuda()
    d_out = torch.empty((N, cfg.param_channels), dtype=torch.float32, device="cuda")
    L = _native.load()
    _native.check(L.lpic_forward_taps(m.handle, d_taps.data_ptr(), N, d_out.data_ptr(), _native.stream_ptr()),
                  "lpic_forward_taps")
    out[:] = d_out.cpu().numpy()
    return out


def forward_full(image_n: np.ndarray, w: Weights, cfg: ModelConfig) -> np.ndarray:
    """Whole-plane network pass (H, W, 3) f32 -> (H, W, M) f32 on the GPU."""
    import torch
    check_weights(w, cfg)
    if image_n.dtype != np.float32 or image_n.ndim != 3 or image_n.shape[2] != 3:
        raise ValueError("expected a normalized HxWx3 float32 plane")
    H, W, _ = image_n.shape
    m = gpu_model(w, cfg)
    d_plane = torch.from_numpy(np.ascontiguousarray(image_n)).cuda()
    d_out = torch.empty((H, W, cfg.param_channels), dtype=torch.float32, device="cuda")
    L = _native.load()
    _native.check(L.lpic_forward_full(m.handle, d_plane.data_ptr(), H, W, d_out.data_ptr(), _native.stream_ptr()),
                  "lpic_forward_full")
    return d_out.cpu().numpy()


def forward_taps_batch(tap_values: np.ndarray, w: Weights, cfg: ModelConfig) -> np.ndarray:
    """(N, T, 3) gathered taps -> (N, M) raw parameters on the GPU."""
    check_weights(w, cfg)
    if tap_values.ndim != 3 or tap_values.shape[1:] != (cfg.tap_count, 3):
        raise ValueError(f"expected (N, {cfg.tap_count}, 3) tap values")
    return _kernel_call_taps(tap_values, w, cfg)


def forward_patch(patch: np.ndarray, w: Weights, cfg: ModelConfig) -> np.ndarray:
    h = cfg.kernel_half
    k = 2 * h + 1
    if patch.shape != (k, k, 3):
        raise ValueError(f"expected a {k}x{k}x3 patch")
    taps = causal_taps(h)
    tv = np.ascontiguousarray(patch[taps[:, 0] + h, taps[:, 1] + h, :], dtype=np.float32)
    return forward_taps_batch(tv[None], w, cfg)[0]


def forward_fc(context: np.ndarray, w: Weights, cfg: ModelConfig) -> np.ndarray:
    check_weights(w, cfg)
    n = 3 * cfg.tap_count
    context = np.ascontiguousarray(context, dtype=np.float32)
    if context.shape != (n,):
        raise ValueError(f"expected a context vector of length {n}")
    return _kernel_call_taps(context.reshape(1, cfg.tap_count, 3), w, cfg)[0]
