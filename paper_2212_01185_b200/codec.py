"""encode / decode and the LPIC container -- the drop-in codec surface.

Mirror of /root/reference/pkg/src/lpic/codec.py (same names, arguments,
exceptions and byte format).  All per-pixel work runs on the B200 through
liblpic_b200.so:

  encode -> k_encode (gather + network + 3 quantised tables per pixel, in
            coding order) + k_rc_encode (one range-coder lane per image)
  decode -> k_decode (persistent wavefront decoder, one CTA per image)

Python does what the reference does around the kernels: argument checks,
the fingerprint gate, container packing and exception mapping.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native, network
from .errors import CorruptStreamError, FingerprintMismatchError, LpicError
from .network import ModelConfig, Weights
from .schedules import ScheduleMode, nonempty_step_count, parse_mode

CONTAINER_MAGIC = b"LPIC"
CONTAINER_VERSION = 1
_HEADER = struct.Struct("<4sBBBBIIQQ")   # codec.py:27 of the reference


@dataclass
class Container:
    mode: ScheduleMode
    mixtures: int
    distribution: int
    width: int
    height: int
    weight_fingerprint: int
    payload: bytes
    version: int = CONTAINER_VERSION

    def to_bytes(self) -> bytes:
        return _HEADER.pack(CONTAINER_MAGIC, self.version, int(self.mode), self.mixtures, self.distribution,
                            self.width, self.height, self.weight_fingerprint, len(self.payload)) + self.payload

    @classmethod
    def from_bytes(cls, data: bytes) -> "Container":
        if len(data) < _HEADER.size or data[:4] != CONTAINER_MAGIC:
            raise LpicError("not a compressed image container")
        _, version, mode, K, dist, width, height, fp, n = _HEADER.unpack(data[:_HEADER.size])
        if version != CONTAINER_VERSION:
            raise LpicError(f"unsupported container version {version}")
        payload = data[_HEADER.size:]
        if len(payload) != n:
            raise LpicError("container payload length mismatch")
        return cls(ScheduleMode(mode), K, dist, width, height, fp, payload, version)


@dataclass
class CodecTrace:
    raw: np.ndarray | None = None     # (N, M) float32, coding order
    cdfs: np.ndarray | None = None    # (N, 3, 257) int64
    order: list = field(default_factory=list)
    network_passes: int = 0


def _check_image(image: np.ndarray) -> None:
    if not isinstance(image, np.ndarray) or image.ndim != 3 or image.shape[2] != 3 or image.dtype != np.uint8:
        raise ValueError("expected an HxWx3 uint8 image")
    if image.shape[0] < 1 or image.shape[1] < 1:
        raise ValueError("empty image")


def _check_mode(mode: ScheduleMode, cfg: ModelConfig) -> None:
    if mode == ScheduleMode.DIAGONAL and cfg.kernel_half != 2:
        raise ValueError("diagonal schedule is only defined for kernel_half=2")


def coding_order(mode, H: int, W: int, kernel_half: int) -> np.ndarray:
    """(N, 2) pixel coordinates in bitstream order (codec.py:111-113)."""
    mode = parse_mode(mode)
    a = W if mode == ScheduleMode.SEQUENTIAL else (kernel_half + 1 if mode == ScheduleMode.WAVEFRONT else 1)
    ii, jj = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    step = (a * ii + jj).reshape(-1)
    idx = np.lexsort((ii.reshape(-1), step))
    return np.stack([ii.reshape(-1)[idx], jj.reshape(-1)[idx]], axis=1).astype(np.int64)


def _passes(mode: ScheduleMode, H: int, W: int, cfg: ModelConfig, encoder: bool) -> int:
    if encoder and mode != ScheduleMode.DIAGONAL:
        return 1          # one whole-image pass (codec.py:125-128)
    return nonempty_step_count(mode, H, W, cfg.kernel_half)


def _fill_trace(trace: CodecTrace, raw, cdf, mode, H, W, cfg, encoder):
    trace.raw = raw
    trace.cdfs = cdf.astype(np.int64)
    trace.order = [tuple(int(v) for v in p) for p in coding_order(mode, H, W, cfg.kernel_half)]
    trace.network_passes = _passes(mode, H, W, cfg, encoder)


def _encode_group(images: np.ndarray, w: Weights, cfg: ModelConfig, mode: ScheduleMode,
                  trace: CodecTrace | None):
    """images (n, H, W, 3) uint8 -> list of payload bytes (one stream each)."""
    n, H, W, _ = images.shape
    m = network.gpu_model(w, cfg)
    L = _native.load()
    if trace is None:
        N = H * W
        cap = n * (6 * N + 64)
        buf = np.empty(cap, np.uint8)
        offs = np.zeros(n, np.int64)
        lens = np.zeros(n, np.int64)
        status = np.zeros(n, np.int32)
        imgs = np.ascontiguousarray(images)
        with m.lock:
            _native.check(L.lpic_encode_batch(m.handle, imgs.ctypes.data, n, H, W, int(mode), buf.ctypes.data, cap,
                                              offs.ctypes.data, lens.ctypes.data, status.ctypes.data,
                                              _native.stream_ptr()), "lpic_encode_batch")
        if np.any(status & _native.LPIC_S_NONFINITE):
            raise LpicError("network produced non-finite parameters")
        if np.any(status):
            raise LpicError(f"encoder status {status.tolist()}")
        return [buf[offs[b]:offs[b] + lens[b]].tobytes() for b in range(n)]
    import torch
    assert n == 1
    N = H * W
    cap = 6 * N + 64
    d_img = torch.from_numpy(np.ascontiguousarray(images)).cuda()
    d_pay = torch.empty(cap, dtype=torch.uint8, device="cuda")
    d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
    d_st = torch.zeros(1, dtype=torch.int32, device="cuda")
    d_raw = torch.empty((N, cfg.param_channels), dtype=torch.float32, device="cuda")
    d_cdf = torch.empty((N, 3, 257), dtype=torch.int32, device="cuda")
    with m.lock:
        _native.check(L.lpic_encode_batch_device(m.handle, d_img.data_ptr(), 1, H, W, int(mode), d_pay.data_ptr(),
                                                 cap, d_len.data_ptr(), d_st.data_ptr(), d_raw.data_ptr(),
                                                 d_cdf.data_ptr(), _native.stream_ptr()), "lpic_encode_batch_device")
    torch.cuda.synchronize()
    st = int(d_st.item())
    if st & _native.LPIC_S_NONFINITE:
        raise LpicError("network produced non-finite parameters")
    if st:
        raise LpicError(f"encoder status {st}")
    ln = int(d_len.item())
    _fill_trace(trace, d_raw.cpu().numpy(), d_cdf.cpu().numpy(), mode, H, W, cfg, True)
    return [d_pay[:ln].cpu().numpy().tobytes()]


def encode(image: np.ndarray, w: Weights, cfg: ModelConfig, mode, trace: CodecTrace | None = None) -> Container:
    """Compress an image on the GPU; losslessly invertible by ``decode``."""
    _check_image(image)
    network.check_weights(w, cfg)
    mode = parse_mode(mode)
    _check_mode(mode, cfg)
    H, W, _ = image.shape
    payload = _encode_group(image[None], w, cfg, mode, trace)[0]
    return Container(mode, cfg.mixtures, int(cfg.distribution), W, H, network.container_fingerprint(w, cfg), payload)


def _on_devices(n: int, devices, fn) -> list:
    """Run fn(lo, hi) -> list over contiguous slices of n items, one host
    thread per device (shard.split_for_devices); the slices' results are
    concatenated in order.  The C-ABI calls release the GIL, so the devices
    work concurrently.  devices=None: the current device only."""
    if devices is None or len(devices) <= 1:
        if devices:
            import torch
            with torch.cuda.device(int(devices[0])):
                return fn(0, n)
        return fn(0, n)
    import threading

    import torch
    from . import shard
    parts = shard.split_for_devices(n, [int(d) for d in devices])
    out: list = [None] * len(parts)
    errs: list = []

    def work(k, d, lo, hi):
        try:
            torch.cuda.set_device(d)
            out[k] = fn(lo, hi)
        except BaseException as e:        # re-raised on the caller's thread
            errs.append(e)

    ts = [threading.Thread(target=work, args=(k, d, lo, hi)) for k, (d, lo, hi) in enumerate(parts)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return [x for part in out for x in part]


def encode_batch(images, w: Weights, cfg: ModelConfig, mode, devices=None) -> list:
    """Encode many images; same-size images share one batched launch.
    devices: optional list of CUDA device indices -- the batch is split into
    contiguous slices, one per device, coded concurrently."""
    network.check_weights(w, cfg)
    mode = parse_mode(mode)
    _check_mode(mode, cfg)
    images = list(images)
    for im in images:
        _check_image(im)
    if devices:
        return _on_devices(len(images), devices, lambda lo, hi: encode_batch(images[lo:hi], w, cfg, mode))
    fp = network.container_fingerprint(w, cfg)
    out: list = [None] * len(images)
    groups: dict = {}
    for k, im in enumerate(images):
        groups.setdefault(im.shape, []).append(k)
    for shape, idx in groups.items():
        pays = _encode_group(np.stack([images[k] for k in idx]), w, cfg, mode, None)
        for k, p in zip(idx, pays):
            out[k] = Container(mode, cfg.mixtures, int(cfg.distribution), shape[1], shape[0], fp, p)
    return out


def _check_container(container: Container, w: Weights, cfg: ModelConfig, fp: int) -> None:
    if container.weight_fingerprint != fp:
        other = "fast" if network.get_precision() == "compat" else "compat"
        if container.weight_fingerprint == network.container_fingerprint(w, cfg, other):
            raise FingerprintMismatchError(
                f"container was encoded in {other} precision; decode it with set_precision({other!r})")
        raise FingerprintMismatchError("container was encoded with different weights")
    if container.mixtures != cfg.mixtures or container.distribution != int(cfg.distribution):
        raise LpicError("container model header does not match the config")


def _decode_group(conts: list, w: Weights, cfg: ModelConfig, trace: CodecTrace | None) -> list:
    H, W, mode = conts[0].height, conts[0].width, ScheduleMode(conts[0].mode)
    _check_mode(mode, cfg)
    n = len(conts)
    m = network.gpu_model(w, cfg)
    L = _native.load()
    lens = np.array([len(c.payload) for c in conts], np.int64)
    offs = np.zeros(n, np.int64)
    offs[1:] = np.cumsum(lens)[:-1]
    blob = np.frombuffer(b"".join(c.payload for c in conts) + b"\0" * 8, np.uint8).copy()
    if trace is None:
        imgs = np.empty((n, H, W, 3), np.uint8)
        status = np.zeros(n, np.int32)
        with m.lock:
            _native.check(L.lpic_decode_batch(m.handle, blob.ctypes.data, offs.ctypes.data, lens.ctypes.data, n, H, W,
                                              int(mode), imgs.ctypes.data, status.ctypes.data, _native.stream_ptr()),
                          "lpic_decode_batch")
        if np.any(status & _native.LPIC_S_CORRUPT):
            raise CorruptStreamError("compressed stream exhausted prematurely")
        return list(imgs)
    import torch
    N = H * W
    d_blob = torch.from_numpy(blob).cuda()
    d_offs = torch.from_numpy(offs).cuda()
    d_lens = torch.from_numpy(lens).cuda()
    d_img = torch.empty((1, H, W, 3), dtype=torch.uint8, device="cuda")
    d_st = torch.zeros(1, dtype=torch.int32, device="cuda")
    d_raw = torch.zeros((N, cfg.param_channels), dtype=torch.float32, device="cuda")
    d_cdf = torch.zeros((N, 3, 257), dtype=torch.int32, device="cuda")
    with m.lock:
        _native.check(L.lpic_decode_batch_device(m.handle, d_blob.data_ptr(), d_offs.data_ptr(), d_lens.data_ptr(), 1,
                                                 H, W, int(mode), d_img.data_ptr(), d_st.data_ptr(), d_raw.data_ptr(),
                                                 d_cdf.data_ptr(), _native.stream_ptr()), "lpic_decode_batch_device")
    torch.cuda.synchronize()
    if int(d_st.item()) & _native.LPIC_S_CORRUPT:
        raise CorruptStreamError("compressed stream exhausted prematurely")
    _fill_trace(trace, d_raw.cpu().numpy(), d_cdf.cpu().numpy(), mode, H, W, cfg, False)
    return [d_img[0].cpu().numpy()]


def decode(container: Container, w: Weights, cfg: ModelConfig, trace: CodecTrace | None = None) -> np.ndarray:
    """Reconstruct the exact image from a container on the GPU."""
    network.check_weights(w, cfg)
    _check_container(container, w, cfg, network.container_fingerprint(w, cfg))
    return _decode_group([container], w, cfg, trace)[0]


def decode_batch(containers, w: Weights, cfg: ModelConfig, devices=None) -> list:
    """Decode many containers; same-geometry streams share one launch (one
    decoder cluster per stream).  devices: as in ``encode_batch``."""
    network.check_weights(w, cfg)
    fp = network.container_fingerprint(w, cfg)
    containers = list(containers)
    for c in containers:
        _check_container(c, w, cfg, fp)
    if devices:
        return _on_devices(len(containers), devices, lambda lo, hi: decode_batch(containers[lo:hi], w, cfg))
    out: list = [None] * len(containers)
    groups: dict = {}
    for k, c in enumerate(containers):
        groups.setdefault((c.height, c.width, int(c.mode)), []).append(k)
    for _, idx in groups.items():
        imgs = _decode_group([containers[k] for k in idx], w, cfg, None)
        for k, im in zip(idx, imgs):
            out[k] = im
    return out


def bpsp(container: Container) -> float:
    return 8.0 * len(container.payload) / (3.0 * container.height * container.width)


def theoretical_bpsp(image: np.ndarray, w: Weights, cfg: ModelConfig, mode=ScheduleMode.SEQUENTIAL) -> float:
    """Mean ideal code length, -log2 P(r,g,b | context) per sub-pixel, with
    the unquantised mixture probabilities the encoder sees (codec.py:255-274
    of the reference; kernels.true_symbol_probs, kernels.py:316-346).  The
    per-sub-pixel terms are computed on the GPU and summed here in coding
    order like the reference's numpy sum."""
    import torch
    _check_image(image)
    network.check_weights(w, cfg)
    mode = parse_mode(mode)
    _check_mode(mode, cfg)
    H, W, _ = image.shape
    m = network.gpu_model(w, cfg)
    L = _native.load()
    d_img = torch.from_numpy(np.ascontiguousarray(image)[None]).cuda()
    d_bits = torch.empty((H * W, 3), dtype=torch.float64, device="cuda")
    with m.lock:
        _native.check(L.lpic_theoretical_bits(m.handle, d_img.data_ptr(), 1, H, W, int(mode), d_bits.data_ptr(),
                                              _native.stream_ptr()), "lpic_theoretical_bits")
    bits = d_bits.cpu().numpy()
    return float(bits.sum() / (3.0 * H * W))


def true_symbol_probs(raw: np.ndarray, syms: np.ndarray, rn: np.ndarray, gn: np.ndarray, K: int, dist: int) -> np.ndarray:
    """kernels.true_symbol_probs on the GPU: raw (N, 12K) f32, syms (N, 3)
    int, rn/gn (N) f32 -> (N, 3) float64."""
    import torch
    _native.require_cuda()
    L = _native.load()
    raw = np.ascontiguousarray(raw, np.float32)
    N, M = raw.shape
    d_raw = torch.from_numpy(raw).cuda()
    d_s = torch.from_numpy(np.ascontiguousarray(syms, np.int64)).cuda()
    d_rn = torch.from_numpy(np.ascontiguousarray(rn, np.float32)).cuda()
    d_gn = torch.from_numpy(np.ascontiguousarray(gn, np.float32)).cuda()
    d_out = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    _native.check(L.lpic_true_symbol_probs(d_raw.data_ptr(), N, M, K, int(dist), d_s.data_ptr(), d_rn.data_ptr(),
                                           d_gn.data_ptr(), d_out.data_ptr(), _native.stream_ptr()),
                  "lpic_true_symbol_probs")
    return d_out.cpu().numpy()
