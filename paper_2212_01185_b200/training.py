"""Desk-scale training on the GPU.

Same API and semantics as the reference trainer
(/root/reference/pkg/src/lpic/training.py): `TrainConfig`, `learning_rate`,
`zero_gradients`, `loss`, `backward`, `Adam`, `train`, `EpochStats`,
`write_curve`.  The loss is the mean over pixels of -log2 P(r, g, b | context)
with teacher forcing (training.py:138-213); the network runs in float32.

Where the work runs:

* the discretised-mixture likelihood and its gradient with respect to the raw
  network outputs -- per pixel 3K components x 2 CDF/PDF evaluations in
  float64, the transcendental-heavy part -- is one fused CUDA kernel
  (`lpic_mixture_loss_grad`, csrc/lpic_train.cu);
* the network forward/backward (training.py:93-129) are plain GEMMs on
  device-resident weights (cuBLAS through torch.matmul, TF32 off: float32
  products like the reference's BLAS);
* Adam keeps its moments on the device; weights are copied back to numpy
  Weights only when a call returns.

Like the reference, the GEMM summation order differs from the codec's
canonical scalar order; only the codec needs bit reproducibility.  Parity:
tests/test_gpu_parity.py compares loss and gradients with the reference's
own `backward` (fixtures from oracle/gen_golden_train.py).
"""

from __future__ import annotations

import csv
import math
import os
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import LpicError
from .network import ModelConfig, Weights, causal_taps, glorot_weights, weight_shapes

LN2 = math.log(2.0)


@dataclass
class TrainConfig:
    batch_size: int = 64
    crop: int = 64
    lr: float = 1e-4
    lr_decay: float = 0.99
    lr_decay_every: int = 5
    epochs: int = 10
    seed: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def __post_init__(self):
        if self.lr <= 0:
            raise ValueError("learning rate must be positive")
        if self.batch_size < 1 or self.crop < 1 or self.epochs < 0:
            raise ValueError("invalid training configuration")


class GradientSet(Weights):
    """One tensor per weight tensor, same shapes."""


def zero_gradients(cfg: ModelConfig, dtype=np.float32) -> GradientSet:
    return GradientSet(*[np.zeros(shape, dtype) for _, shape in weight_shapes(cfg)])


def learning_rate(tc: TrainConfig, epoch: int) -> float:
    return tc.lr * tc.lr_decay ** (epoch // tc.lr_decay_every)


@contextmanager
def _fp32_gemms():
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def _float_type(dtype):
    """numpy float32 / float64 -> the matching torch dtype (the reference's
    float64 path is the finite-difference oracle)."""
    import torch
    d = np.dtype(dtype)
    if d == np.float32:
        return torch.float32
    if d == np.float64:
        return torch.float64
    raise ValueError("the trainer runs in float32 or float64")


def _device_weights(w: Weights, dtype=np.float32):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(t, dtype)).cuda() for t in w.tensors()]


def _gather_causal(x, taps):
    """(B, H, W, 3) -> (B*H*W, T*3) causal tap values, zero padded
    (training._gather_causal, training.py:69-82)."""
    import torch
    B, H, W, _ = x.shape
    h = int(np.abs(taps).max())
    xp = torch.nn.functional.pad(x, (0, 0, h, h, h, 0))        # rows: h above; cols: h left and right
    cols = [xp[:, h + int(di):h + int(di) + H, h + int(dj):h + int(dj) + W, :] for di, dj in taps]
    return torch.stack(cols, dim=3).reshape(B * H * W, taps.shape[0] * 3)


def _lrelu(z):
    import torch
    return torch.where(z >= 0, z, z * 0.01)


def _forward(x1, dw, cfg: ModelConfig):
    mw, mb, hw, hb, ow, ob = dw
    T, C = cfg.tap_count, cfg.filters
    zs = [x1 @ mw.reshape(T * 3, C) + mb]
    a = _lrelu(zs[0])
    for l in range(cfg.hidden_count):
        z = a @ hw[l].T + hb[l]
        zs.append(z)
        a = _lrelu(z)
    raw = a @ ow.T + ob
    return raw, zs


def _backward(draw, x1, zs, dw, cfg: ModelConfig):
    import torch
    mw, mb, hw, hb, ow, ob = dw
    g = [None] * 6
    a_last = _lrelu(zs[-1])
    g[4] = draw.T @ a_last
    g[5] = draw.sum(dim=0)
    ga = draw @ ow
    gh_w = [None] * cfg.hidden_count
    gh_b = [None] * cfg.hidden_count
    for l in range(cfg.hidden_count - 1, -1, -1):
        gz = ga * torch.where(zs[l + 1] >= 0, 1.0, 0.01)
        a_prev = _lrelu(zs[l])
        gh_w[l] = gz.T @ a_prev
        gh_b[l] = gz.sum(dim=0)
        ga = gz @ hw[l]
    gz = ga * torch.where(zs[0] >= 0, 1.0, 0.01)
    g[0] = (x1.T @ gz).reshape(mw.shape)
    g[1] = gz.sum(dim=0)
    g[2] = torch.stack(gh_w) if cfg.hidden_count else torch.zeros_like(hw)
    g[3] = torch.stack(gh_b) if cfg.hidden_count else torch.zeros_like(hb)
    return g


def _check_batch(batch):
    if not isinstance(batch, np.ndarray) or batch.ndim != 4 or batch.shape[0] < 1 or batch.shape[3] != 3 \
            or batch.dtype != np.uint8:
        raise ValueError("expected a nonempty (B, H, W, 3) uint8 batch")


def _mixture_device(raw, d_pix, cfg: ModelConfig, want_grad: bool):
    """raw (N, 12K) float32/float64 device tensor, d_pix (N, 3) u8 -> (mean
    -log2 p per pixel, d loss / d raw | None), the fused likelihood kernel
    (training._mixture_loss, training.py:138-213)."""
    import torch
    L = _native.require_cuda()
    N = raw.shape[0]
    raw = raw.contiguous()
    logp = torch.empty(N, dtype=torch.float64, device=raw.device)
    draw = torch.empty_like(raw) if want_grad else None
    fn = L.lpic_mixture_loss_grad_f64 if raw.dtype == torch.float64 else L.lpic_mixture_loss_grad
    _native.check(fn(raw.data_ptr(), d_pix.data_ptr(), N, cfg.mixtures, int(cfg.distribution), logp.data_ptr(),
                     draw.data_ptr() if want_grad else None, _native.stream_ptr()), "mixture loss")
    return float(-logp.sum().item() / N / LN2), draw


def _loss_grad_device(d_batch, dw, cfg: ModelConfig, want_grad: bool, dtype=np.float32):
    """Device batch (B, H, W, 3) u8 -> (loss, [6 gradient tensors] | None)."""
    tdt = _float_type(dtype)
    x = d_batch.to(tdt) / 127.5 - 1.0                         # training._normalize_batch
    taps = causal_taps(cfg.kernel_half)
    with _fp32_gemms():
        x1 = _gather_causal(x, taps)
        raw, zs = _forward(x1, dw, cfg)
        value, draw = _mixture_device(raw, d_batch.reshape(-1, 3), cfg, want_grad)
        grads = _backward(draw, x1, zs, dw, cfg) if want_grad else None
    return value, grads


def loss(batch: np.ndarray, w: Weights, cfg: ModelConfig, dtype=np.float32) -> float:
    """Mean -log2 P(r, g, b | context) per pixel over the batch, in bits
    (training.py:219-228); dtype float32 (the trainer) or float64."""
    import torch
    _check_batch(batch)
    value, _ = _loss_grad_device(torch.from_numpy(np.ascontiguousarray(batch)).cuda(), _device_weights(w, dtype),
                                 cfg, False, dtype)
    return value


def backward(batch: np.ndarray, w: Weights, cfg: ModelConfig, dtype=np.float32) -> tuple[float, GradientSet]:
    """Loss plus analytic gradients for every weight tensor (training.py:231-240)."""
    import torch
    _check_batch(batch)
    value, g = _loss_grad_device(torch.from_numpy(np.ascontiguousarray(batch)).cuda(), _device_weights(w, dtype),
                                 cfg, True, dtype)
    return value, GradientSet(*[t.cpu().numpy() for t in g])


# The reference's internal stages, with the same arguments (its tests call
# them): host arrays in and out, the work on the GPU.
def _normalize_batch(images: np.ndarray, dtype):
    x = images.astype(dtype)
    return x / dtype(127.5) - dtype(1.0)


def _network_forward(xn: np.ndarray, w: Weights, cfg: ModelConfig, dtype):
    """(B, H, W, 3) normalised -> raw (B, H, W, M) and the backward cache
    (gathered taps, pre-activations; device tensors)."""
    import torch
    B, H, W, _ = xn.shape
    dw = _device_weights(w, dtype)
    with _fp32_gemms():
        x1 = _gather_causal(torch.from_numpy(np.ascontiguousarray(xn, dtype)).cuda(), causal_taps(cfg.kernel_half))
        raw, zs = _forward(x1, dw, cfg)
    return raw.reshape(B, H, W, cfg.param_channels).cpu().numpy(), (x1, zs)


def _network_backward(draw, cache, w: Weights, cfg: ModelConfig) -> GradientSet:
    import torch
    x1, zs = cache
    dw = _device_weights(w, np.float64 if x1.dtype == torch.float64 else np.float32)
    d = torch.from_numpy(np.ascontiguousarray(draw).reshape(x1.shape[0], cfg.param_channels)).to(x1)
    with _fp32_gemms():
        g = _backward(d, x1, zs, dw, cfg)
    return GradientSet(*[t.cpu().numpy() for t in g])


def _mixture_loss(raw, images, cfg: ModelConfig, want_grad: bool):
    """(loss in bits per pixel, d loss / d raw shaped like raw | None)."""
    import torch
    r = np.ascontiguousarray(raw)
    value, draw = _mixture_device(torch.from_numpy(r.reshape(-1, cfg.param_channels)).cuda(),
                                  torch.from_numpy(np.ascontiguousarray(images, np.uint8).reshape(-1, 3)).cuda(),
                                  cfg, want_grad)
    return value, (draw.cpu().numpy().reshape(r.shape) if want_grad else None)


def finite_difference_check(cfg: ModelConfig | None = None, checks: int = 200, seed: int = 0, eps: float = 1e-3,
                            batch_shape=(2, 8, 8)):
    """Analytic (GPU backward, float64) vs central finite-difference
    gradients at randomly drawn scalar parameters; the reference's check
    (training.py:352-414): randomised biases, draws whose +-eps window
    crosses a LeakyReLU kink are redrawn.  Returns (worst relative error,
    [(tensor, index, analytic, numeric, rel)])."""
    cfg = cfg or ModelConfig(mixtures=2, filters=8, layers=4)
    rng = np.random.default_rng(seed)
    B, H, W = batch_shape
    batch = rng.integers(0, 256, (B, H, W, 3), dtype=np.uint8)
    w32 = glorot_weights(cfg, rng)
    for b in (w32.masked_b, w32.hidden_b, w32.out_b):
        b[:] = rng.uniform(-0.3, 0.3, b.shape)
    w = Weights(*[t.astype(np.float64) for t in w32.tensors()])
    _, grads = backward(batch, w, cfg, dtype=np.float64)
    xn = _normalize_batch(batch, np.float64)

    def at_current():
        raw, (_, zs) = _network_forward(xn, w, cfg, np.float64)
        return _mixture_loss(raw, batch, cfg, want_grad=False)[0], zs

    params, gparams = w.tensors(), grads.tensors()
    records, worst, tries = [], 0.0, 0
    while len(records) < checks:
        tries += 1
        if tries > 50 * checks:
            raise LpicError("gradient check could not find enough kink-free draws")
        ti = int(rng.integers(0, len(params)))
        k = int(rng.integers(0, params[ti].size))
        x0 = float(params[ti].flat[k])
        params[ti].flat[k] = x0 + eps
        up, z_up = at_current()
        params[ti].flat[k] = x0 - eps
        down, z_dn = at_current()
        params[ti].flat[k] = x0
        if any(bool(((a >= 0) != (b >= 0)).any()) for a, b in zip(z_up, z_dn)):
            continue
        numeric = (up - down) / (2.0 * eps)
        analytic = float(gparams[ti].flat[k])
        rel = abs(numeric - analytic) / max(abs(numeric), abs(analytic), 1e-6)
        worst = max(worst, rel)
        records.append((ti, k, analytic, numeric, rel))
    return worst, records


class Adam:
    """Adam with the reference's update (training.py:248-266); moments live on
    the device.  `step` accepts numpy Weights/GradientSet (updated in place)
    like the reference; the trainer uses `step_device`."""

    def __init__(self, cfg: ModelConfig, tc: TrainConfig):
        import torch
        self.tc = tc
        self.m = [torch.zeros(s, dtype=torch.float32, device="cuda") for _, s in weight_shapes(cfg)]
        self.v = [torch.zeros(s, dtype=torch.float32, device="cuda") for _, s in weight_shapes(cfg)]
        self.t = 0

    def step_device(self, dw, dg, lr: float) -> None:
        import torch
        self.t += 1
        b1, b2, eps = self.tc.beta1, self.tc.beta2, self.tc.eps
        c1 = 1.0 - b1 ** self.t
        c2 = 1.0 - b2 ** self.t
        for wt, gt, mt, vt in zip(dw, dg, self.m, self.v):
            mt.mul_(b1).add_((1.0 - b1) * gt)
            vt.mul_(b2).add_((1.0 - b2) * torch.square(gt))
            wt.sub_((lr / c1) * mt / (torch.sqrt(vt / c2) + eps))

    def step(self, w: Weights, g: GradientSet, lr: float) -> None:
        dw = _device_weights(w)
        self.step_device(dw, _device_weights(g), lr)
        for dst, src in zip(w.tensors(), dw):
            dst[...] = src.cpu().numpy()


@dataclass
class EpochStats:
    epoch: int
    loss_bits_per_pixel: float
    bpsp_estimate: float
    lr: float


def _random_crop(image: np.ndarray, crop: int, rng: np.random.Generator):
    H, W, _ = image.shape
    i = int(rng.integers(0, H - crop + 1))
    j = int(rng.integers(0, W - crop + 1))
    return image[i:i + crop, j:j + crop]


def train(images, tc: TrainConfig, cfg: ModelConfig, initial: Weights | None = None, on_epoch=None):
    """Train on shuffled random crops; deterministic batch order given the seed
    (the same crops and permutation as the reference, training.py:288-333).
    Returns (weights, per-epoch stats)."""
    import torch
    if len(images) == 0:
        raise LpicError("empty training dataset")
    if tc.crop < 2 * cfg.kernel_half + 1:
        raise ValueError("crop smaller than the network's receptive field")
    smallest = min(min(im.shape[0], im.shape[1]) for im in images)
    if smallest < tc.crop:
        raise LpicError(f"crop {tc.crop} larger than smallest image ({smallest})")
    rng = np.random.default_rng(tc.seed)
    w = initial.copy() if initial is not None else glorot_weights(cfg, rng)
    dw = _device_weights(w)
    opt = Adam(cfg, tc)
    curve = []
    for epoch in range(tc.epochs):
        lr = learning_rate(tc, epoch)
        perm = rng.permutation(len(images))
        losses = []
        for k in range(0, len(perm), tc.batch_size):
            chunk = perm[k:k + tc.batch_size]
            batch = np.stack([_random_crop(images[i], tc.crop, rng) for i in chunk])
            value, dg = _loss_grad_device(torch.from_numpy(batch).cuda(), dw, cfg, True)
            if not math.isfinite(value):
                raise LpicError(f"non-finite loss at epoch {epoch}, batch {k // tc.batch_size}")
            opt.step_device(dw, dg, lr)
            losses.append(value)
        mean_loss = float(np.mean(losses))
        stats = EpochStats(epoch, mean_loss, mean_loss / 3.0, lr)
        curve.append(stats)
        if on_epoch is not None:
            on_epoch(stats)
    for dst, src in zip(w.tensors(), dw):
        dst[...] = src.cpu().numpy()
    return w, curve


def write_curve(path, curve) -> None:
    with open(path, "w", newline="") as f:
        writer = csv.writer(f)
        writer.writerow(["epoch", "loss_bits_per_pixel", "bpsp_estimate", "lr"])
        for st in curve:
            writer.writerow([st.epoch, repr(st.loss_bits_per_pixel), repr(st.bpsp_estimate), repr(st.lr)])
