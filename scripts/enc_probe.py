"""Device-timed C2 encode (events on the caller's stream), per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import _native, synth
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
H, W = 512, 768
N = H * W
w, cfg = synth.baseline_weights()
imgs = bench.make_images(bench.CONFIGS["c2"], 0, 1, False)[:n]
L = _native.require_cuda()
m = P.network.gpu_model(w, cfg)
st = torch.cuda.Stream(); sp = int(st.cuda_stream)
d_imgs = torch.from_numpy(imgs).cuda()
cap = 6 * N + 64
d_pay = torch.empty(n * cap, dtype=torch.uint8, device="cuda")
d_lens = torch.zeros(n, dtype=torch.int64, device="cuda"); d_st = torch.zeros(n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(5):
    with torch.cuda.stream(st):
        flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    _native.check(L.lpic_encode_batch_device(m.handle, d_imgs.data_ptr(), n, H, W, 1, d_pay.data_ptr(), cap,
                                             d_lens.data_ptr(), d_st.data_ptr(), None, None, sp), "enc")
    e1.record(st); st.synchronize()
    print(f"encode {e0.elapsed_time(e1):.1f} ms  status {int(d_st.sum())}  bytes {int(d_lens.sum())}", flush=True)
