"""Synthetic inputs for the benchmark configs (harness definitions).

The reference has no 1/f generator and no Kaiming init;
these follow the SURVEY 8(d) specification verbatim so CPU and GPU runs see
identical seeded images.  Not on the hot path.
"""

from __future__ import annotations

import numpy as np

from .network import ModelConfig, glorot_weights, kaiming_weights  # noqa: F401  (re-export)


def synth_1f(seed: int, H: int, W: int, beta=None, rho: float = 0.8, sigma=None,
             contrast: float = 40.0) -> np.ndarray:
    """1/f-spectrum RGB image, inter-channel correlation rho, Gaussian noise sigma."""
    rng = np.random.default_rng(seed)
    if beta is None:
        beta = rng.uniform(1.6, 2.4)
    if sigma is None:
        sigma = rng.uniform(2.0, 6.0)
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.rfftfreq(W)[None, :]
    f = np.sqrt(fx ** 2 + fy ** 2)
    f[0, 0] = 1.0
    amp = f ** (-beta / 2.0)
    amp[0, 0] = 0.0

    def field():
        z = rng.standard_normal((H, W))
        x = np.fft.irfft2(np.fft.rfft2(z) * amp, s=(H, W))
        return (x - x.mean()) / (x.std() + 1e-12)

    shared = field()
    chans = [np.sqrt(rho) * shared + np.sqrt(1.0 - rho) * field() for _ in range(3)]
    img = np.stack(chans, axis=2) * contrast + 128.0 + rng.standard_normal((H, W, 3)) * sigma
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def c1_image() -> np.ndarray:
    """BASELINE configs[0]: 64x64, seed 0, beta=2.0, sigma=3."""
    return synth_1f(0, 64, 64, beta=2.0, sigma=3.0)


def batch(n: int, H: int, W: int, seed0: int = 0) -> np.ndarray:
    return np.stack([synth_1f(seed0 + k, H, W) for k in range(n)])


def baseline_weights(cfg: ModelConfig | None = None):
    """'Kaiming seed 0' weights of the reference config."""
    cfg = cfg or ModelConfig()
    return kaiming_weights(cfg, np.random.default_rng(0)), cfg


def synth_1f_gray(seed: int, H: int, W: int, beta=None, sigma=None, contrast: float = 40.0) -> np.ndarray:
    """Single-channel variant (BASELINE configs[4] grayscale): one 1/f field
    plus noise, same draw conventions as synth_1f."""
    rng = np.random.default_rng(seed)
    if beta is None:
        beta = rng.uniform(1.6, 2.4)
    if sigma is None:
        sigma = rng.uniform(2.0, 6.0)
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.rfftfreq(W)[None, :]
    f = np.sqrt(fx ** 2 + fy ** 2)
    f[0, 0] = 1.0
    amp = f ** (-beta / 2.0)
    amp[0, 0] = 0.0
    z = rng.standard_normal((H, W))
    x = np.fft.irfft2(np.fft.rfft2(z) * amp, s=(H, W))
    x = (x - x.mean()) / (x.std() + 1e-12)
    img = x * contrast + 128.0 + rng.standard_normal((H, W)) * sigma
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def fitted_weights(steps: int = 200, seed: int = 0, n_train: int = 64, size: int = 128):
    """BASELINE configs[1]'s optional variant: Kaiming seed 0 weights fitted
    for `steps` steps of the trainer (TrainConfig defaults: batch 64 of 64x64
    crops, Adam lr 1e-4 with its stepped decay) on images of the same 1/f
    generator (seeds 10_000.. -- disjoint from the benchmark images).  Runs on
    the GPU (training.py); deterministic for a given device and library."""
    from . import training
    w, cfg = baseline_weights()
    imgs = list(batch(n_train, size, size, seed0=10_000 + 1000 * seed))
    tc = training.TrainConfig(batch_size=n_train, epochs=steps, seed=seed)   # one batch per epoch
    w, curve = training.train(imgs, tc, cfg, initial=w)
    return w, cfg, curve


def flat_weights(log_scale: float = 7.0):
    """Kaiming seed 0 with every mixture log-scale bias at `log_scale` (e^7:
    the clip limit, network.py / kernels.py:242-247): near-flat PMFs whose
    quantisation remainders mostly share one digit -- the worst case of the
    deficit selection (the "flat-mixture cliff")."""
    w, cfg = baseline_weights()
    K = cfg.mixtures
    w = w.copy()
    w.out_b[6 * K:9 * K] = np.float32(log_scale)
    return w, cfg
