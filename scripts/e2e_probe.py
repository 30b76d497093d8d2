"""Device-resident vs host-buffer (e2e) decode timing on the C2 batch, per call."""
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
h_img = torch.from_numpy(imgs).pin_memory()
cap = 6 * N * n + 64
h_pay = torch.empty(cap, dtype=torch.uint8).pin_memory()
h_offs = np.zeros(n, np.int64); h_lens = np.zeros(n, np.int64); h_st = np.zeros(n, np.int32)
h_out = torch.empty((n, H, W, 3), dtype=torch.uint8).pin_memory()
_native.check(L.lpic_encode_batch(m.handle, h_img.data_ptr(), n, H, W, 1, h_pay.data_ptr(), cap, h_offs.ctypes.data,
                                  h_lens.ctypes.data, h_st.ctypes.data, sp), "enc")
d_pay = torch.from_numpy(h_pay.numpy()).cuda(); d_offs = torch.from_numpy(h_offs).cuda(); d_lens = torch.from_numpy(h_lens).cuda()
d_out = torch.empty((n, H, W, 3), dtype=torch.uint8, device="cuda"); d_st = torch.zeros(n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    _native.check(L.lpic_decode_batch_device(m.handle, d_pay.data_ptr(), d_offs.data_ptr(), d_lens.data_ptr(), n, H, W, 1,
                                             d_out.data_ptr(), d_st.data_ptr(), None, None, sp), "dec")
    e1.record(st); st.synchronize()
    print(f"device: {e0.elapsed_time(e1):.1f} ms (wall {1e3*(time.perf_counter()-t0):.1f})", flush=True)
    t0 = time.perf_counter()
    _native.check(L.lpic_decode_batch(m.handle, h_pay.data_ptr(), h_offs.ctypes.data, h_lens.ctypes.data, n, H, W, 1,
                                      h_out.data_ptr(), h_st.ctypes.data, sp), "dec e2e")
    print(f"e2e: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
assert torch.equal(h_out, h_img)
