"""Decoder timeline: producer chunk / consumer pixel timestamps for stream 0.
Needs a timeline build: python scripts/ab_build.py tl --all -DLPIC_DEC_TIMELINE
(+ -DLPIC_DEC_PROF for the in-situ chain phases), run with LPIC_LIB=.../ab/tl.so."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import _native, synth
H = int(sys.argv[1]) if len(sys.argv) > 1 else 128
W = int(sys.argv[2]) if len(sys.argv) > 2 else H
NI = int(sys.argv[3]) if len(sys.argv) > 3 else 1      # streams decoded concurrently (stream 0 is traced)
if os.environ.get("LPIC_PRECISION"):
    P.set_precision(os.environ["LPIC_PRECISION"])     # compat (default) or fast
w, cfg = synth.baseline_weights()
imgs = synth.batch(NI, H, W)
cs = P.encode_batch(imgs, w, cfg, "wave")
m = P.network.gpu_model(w, cfg)
L = _native.load()
L.lpic_decode_debug.argtypes = [C.c_void_p, C.c_void_p]
P.decode_batch(cs, w, cfg)                          # builds the geometry tables
nch = L.lpic_decode_debug(m.handle, None)
N = H * W
buf = torch.zeros(4 * nch + 12 * N + 16, dtype=torch.int64, device="cuda")
L.lpic_decode_debug(m.handle, buf.data_ptr())
out = P.decode_batch(cs, w, cfg)
L.lpic_decode_debug(m.handle, None)
assert all(np.array_equal(o, i) for o, i in zip(out, imgs))
b = buf.cpu().numpy().astype(np.float64)
t0 = min(b[:4 * nch][b[:4 * nch] > 0].min(), b[4 * nch:4 * nch + 12 * N].reshape(-1, 12)[:, 0].min())
pc = (b[:4 * nch].reshape(nch, 4) - t0) / 1e3     # us
raw12 = b[4 * nch:4 * nch + 12 * N].reshape(N, 12)
prof = b[4 * nch + 12 * N:]
cp = (raw12[:, :3] - t0) / 1e3
clk = raw12[:, 3:10]
print(f"total {cp[-1, 2]:.1f} us for {N} px ({cp[-1,2]/N:.2f} us/px), {nch} chunks")
print("producer: wait %.1f us/chunk, net+mix %.1f, tables %.1f (means)" % (
    np.mean(pc[:, 1] - pc[:, 0]), np.mean(pc[:, 2] - pc[:, 1]), np.mean(pc[:, 3] - pc[:, 2])))
print("consumer: full-wait %.2f us/px, chain %.2f us/px" % (np.mean(cp[:, 1] - cp[:, 0]), np.mean(cp[:, 2] - cp[:, 1])))
np.save("gpurun_out/timeline.npy", b)
mid = clk[N // 4: 3 * N // 4]
print("chain phases (cycles/px): red-search %.0f green-pmf %.0f green-quant %.0f green-dec+blue-pmf %.0f blue-quant %.0f "
      "blue-dec+write %.0f" % tuple(np.mean(np.diff(mid, axis=1), axis=0)))
print("chain total cycles/px %.0f" % np.mean(mid[:, -1] - mid[:, 0]))
for k in list(range(0, min(nch, 12))) + list(range(nch // 2, nch // 2 + 6)):
    print("chunk", k, np.round(pc[k], 1))
for n in list(range(0, 6)) + list(range(N // 2, N // 2 + 6)):
    print("px", n, np.round(cp[n], 1))
print("raw consumer rows", raw12[N // 2].astype(np.int64), raw12[N // 2 + 1].astype(np.int64))
nz = np.nonzero(raw12[:, 0])[0]
print("nonzero consumer rows:", len(nz), nz[:5], nz[-5:] if len(nz) else None)
if prof.any():
    nm = ["P cdf", "bar E", "pmf+fx", "bar T", "Q rest", "bar A", "S level2+", "prefix", "-", "D search", "Q scale",
          "P z", "P phi", "S level1"]
    print("in-situ chain phases (cycles per table, stream 0, %d tables):" % (2 * N))
    for i in range(14):
        print("  %-10s %6.0f" % (nm[i], prof[i] / (2 * N)))
