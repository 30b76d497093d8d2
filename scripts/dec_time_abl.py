"""(Ablation variant of dec_time.py: decode status and losslessness are NOT
checked, so ABL_* builds -- which decode garbage on purpose -- can be timed.)
Device-resident C2 decode time (CUDA events, L2 flushed between reps),
median over reps.  LPIC_LIB selects an A/B build.
usage: python scripts/dec_time.py [kaiming|fitted|flat] [reps] [n_images]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import _native, synth
kind = sys.argv[1] if len(sys.argv) > 1 else "kaiming"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(sys.argv[3]) if len(sys.argv) > 3 else 24
w, cfg = synth.baseline_weights()
if kind == "fitted":
    w, cfg, _ = synth.fitted_weights()
elif kind == "flat":
    w, cfg = synth.flat_weights()
H, W = 512, 768
imgs = synth.batch(n, H, W)
L = _native.load()
m = P.network.gpu_model(w, cfg)
d_imgs = torch.from_numpy(imgs).cuda()
cap = 6 * H * W + 64
d_pay = torch.empty(n * cap, dtype=torch.uint8, device="cuda")
d_lens = torch.zeros(n, dtype=torch.int64, device="cuda")
d_st = torch.zeros(n, dtype=torch.int32, device="cuda")
d_out = torch.empty((n, H, W, 3), dtype=torch.uint8, device="cuda")
d_offs = torch.arange(n, dtype=torch.int64, device="cuda") * cap
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
_native.check(L.lpic_encode_batch_device(m.handle, d_imgs.data_ptr(), n, H, W, 1, d_pay.data_ptr(), cap,
                                         d_lens.data_ptr(), d_st.data_ptr(), None, None, s), "enc")
ms = []
for r in range(reps + 1):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.lpic_decode_batch_device(m.handle, d_pay.data_ptr(), d_offs.data_ptr(), d_lens.data_ptr(), n, H,
                               W, 1, d_out.data_ptr(), d_st.data_ptr(), None, None, s)
    e1.record(); torch.cuda.synchronize()
    if r >= 1:
        ms.append(e0.elapsed_time(e1))
print("lossless", torch.equal(d_out, d_imgs))
med = statistics.median(ms)
print(f"{os.path.basename(os.environ.get('LPIC_LIB', 'main'))} {kind} n={n}: decode {med:.1f} ms "
      f"({3 * H * W * n / med / 1e3:.2f} Msubpx/s)")
