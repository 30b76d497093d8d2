"""GPU training step throughput (TrainConfig defaults: batch 64 of 64x64 crops,
the reference network K=3 C=128 L=5): loss + backward + Adam, device-resident
weights, events on the current stream.  Also times the fused mixture-loss
kernel alone."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_01185_b200 import training, synth, _native
from paper_2212_01185_b200.network import ModelConfig, glorot_weights
cfg = ModelConfig()
tc = training.TrainConfig()
rng = np.random.default_rng(0)
w = glorot_weights(cfg, rng)
imgs = synth.batch(8, 256, 256)
dw = training._device_weights(w)
opt = training.Adam(cfg, tc)
B, crop = tc.batch_size, tc.crop

def batch():
    return np.stack([training._random_crop(imgs[int(rng.integers(0, len(imgs)))], crop, rng) for _ in range(B)])

batches = [torch.from_numpy(batch()).cuda() for _ in range(8)]
for k in range(3):
    v, g = training._loss_grad_device(batches[k], dw, cfg, True); opt.step_device(dw, g, tc.lr)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 20
e0.record()
for k in range(steps):
    v, g = training._loss_grad_device(batches[k % 8], dw, cfg, True)
    opt.step_device(dw, g, tc.lr)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
px = B * crop * crop
print(f"train step {ms:.2f} ms  ({px / ms / 1e3:.2f} Mpixel/s, loss {v:.4f} bits/px)")
# the fused likelihood kernel alone
L = _native.load()
N = px
raw = torch.randn(N, 36, device="cuda") * 0.5
d = batches[0].reshape(N, 3).contiguous()
logp = torch.empty(N, dtype=torch.float64, device="cuda"); draw = torch.empty_like(raw)
for _ in range(3):
    L.lpic_mixture_loss_grad(raw.data_ptr(), d.data_ptr(), N, 3, 0, logp.data_ptr(), draw.data_ptr(), _native.stream_ptr())
torch.cuda.synchronize(); e0.record()
for _ in range(20):
    L.lpic_mixture_loss_grad(raw.data_ptr(), d.data_ptr(), N, 3, 0, logp.data_ptr(), draw.data_ptr(), _native.stream_ptr())
e1.record(); torch.cuda.synchronize()
print(f"mixture loss+grad kernel {e0.elapsed_time(e1) / 20:.3f} ms for {N} px")
