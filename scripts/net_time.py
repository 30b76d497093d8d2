"""FAST encoder network (k_enc_net_tc2) alone on C2 (24 x 768x512): median
ms over reps through lpic_network_coding_order (LPIC_LIB selects an A/B build)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import _native, synth
w, cfg = synth.baseline_weights()
P.set_precision("fast")
H, W, n = 512, 768, 24
imgs = synth.batch(n, H, W)
L = _native.load()
m = P.network.gpu_model(w, cfg)
d_imgs = torch.from_numpy(imgs).cuda()
raw = torch.empty((n, H * W, 36), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
ms = []
for r in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.lpic_network_coding_order(m.handle, d_imgs.data_ptr(), n, H, W, 1, raw.data_ptr(), st)
    e1.record(); torch.cuda.synchronize()
    if r >= 1:
        ms.append(e0.elapsed_time(e1))
med = statistics.median(ms)
print(f"{os.path.basename(os.environ.get('LPIC_LIB', 'main'))}: network {med:.3f} ms, "
      f"{n * H * W * 3 * 38912 / med / 1e9:.1f} model TFLOP/s")
