"""Device-resident C2 encode time (CUDA events, L2 flushed between reps):
median ms over reps.  LPIC_LIB selects an A/B build.
usage: python scripts/enc_time.py [kaiming|fitted|flat] [reps] [fast]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import _native, synth
kind = sys.argv[1] if len(sys.argv) > 1 else "kaiming"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w, cfg = synth.baseline_weights()
if kind == "fitted":
    w, cfg, _ = synth.fitted_weights()
elif kind == "flat":
    w, cfg = synth.flat_weights()
if "fast" in sys.argv:
    P.set_precision("fast")
H, W, n = 512, 768, 24
imgs = synth.batch(n, H, W)
L = _native.load()
m = P.network.gpu_model(w, cfg)
d_imgs = torch.from_numpy(imgs).cuda()
cap = 6 * H * W + 64
d_pay = torch.empty(n * cap, dtype=torch.uint8, device="cuda")
d_lens = torch.zeros(n, dtype=torch.int64, device="cuda")
d_st = torch.zeros(n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
ms = []
for r in range(reps + 2):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.check(L.lpic_encode_batch_device(m.handle, d_imgs.data_ptr(), n, H, W, 1, d_pay.data_ptr(), cap,
                                             d_lens.data_ptr(), d_st.data_ptr(), None, None, st.cuda_stream), "enc")
    e1.record(); torch.cuda.synchronize()
    if r >= 2:
        ms.append(e0.elapsed_time(e1))
tot = int(d_lens.sum())
print(f"{os.path.basename(os.environ.get('LPIC_LIB', 'main'))} {kind}: encode {statistics.median(ms):.2f} ms "
      f"({3 * H * W * n / statistics.median(ms) / 1e3:.1f} Msubpx/s) bytes {tot}")
