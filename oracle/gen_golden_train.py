"""Reference loss / gradients / short training runs of the desk-scale trainer
(training.py:93-333), written to tests/golden/reference_train.npz.  Runs the
REFERENCE package read-only in this container (like gen_golden.py):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_train.py

Cases: (tiny: K=2 C=8 L=4, Gaussian), (small_logistic: K=3 C=16 L=5,
Logistic), (ref: K=3 C=128 L=5, Gaussian); random uint8 batches with some
saturated pixels (0 / 255 exercise the +-inf bin edges); glorot weights with
random biases.  Plus a 2-epoch `train` run on four 24x24 images.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from lpic import training  # noqa: E402  (the reference)
from lpic.network import Distribution, ModelConfig, glorot_weights  # noqa: E402

OUT = os.path.join(HERE, "..", "tests", "golden", "reference_train.npz")
CFGS = {
    "tiny": ModelConfig(mixtures=2, filters=8, layers=4),
    "small_logistic": ModelConfig(mixtures=3, filters=16, layers=5, distribution=Distribution.LOGISTIC),
    "ref": ModelConfig(),
}
NAMES = ["masked_w", "masked_b", "hidden_w", "hidden_b", "out_w", "out_b"]


def main():
    out = {}
    for idx, (name, cfg) in enumerate(CFGS.items()):
        rng = np.random.default_rng(100 + idx)
        batch = rng.integers(0, 256, (2, 12, 10, 3), dtype=np.uint8)
        batch[0, :2, :3] = 0
        batch[1, -2:, -3:] = 255
        w = glorot_weights(cfg, rng)
        w.masked_b[:] = rng.uniform(-0.3, 0.3, w.masked_b.shape)
        w.hidden_b[:] = rng.uniform(-0.3, 0.3, w.hidden_b.shape)
        w.out_b[:] = rng.uniform(-0.3, 0.3, w.out_b.shape)
        value, g = training.backward(batch, w, cfg)
        out[f"{name}_batch"] = batch
        for n, t in zip(NAMES, w.tensors()):
            out[f"{name}_w_{n}"] = t
        for n, t in zip(NAMES, g.tensors()):
            out[f"{name}_g_{n}"] = t
        out[f"{name}_loss"] = np.float64(value)
        print(name, value)
    # a short training run (tiny config)
    rng = np.random.default_rng(7)
    imgs = [rng.integers(0, 256, (24, 24, 3), dtype=np.uint8) for _ in range(4)]
    tc = training.TrainConfig(batch_size=2, crop=16, lr=1e-3, epochs=2, seed=3)
    w, curve = training.train(imgs, tc, CFGS["tiny"])
    out["run_images"] = np.stack(imgs)
    out["run_curve"] = np.array([s.loss_bits_per_pixel for s in curve])
    for n, t in zip(NAMES, w.tensors()):
        out[f"run_w_{n}"] = t
    print("run", out["run_curve"])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
