"""C2 encode + decode once through the device C-ABI (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import _native, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
H, W = 512, 768
w, cfg = synth.baseline_weights()
if os.environ.get("FITTED"):
    w, cfg, _ = synth.fitted_weights()
imgs = synth.batch(n, H, W)
cs = P.encode_batch(imgs, w, cfg, "wave")
if "--decode" in sys.argv:
    out = P.decode_batch(cs, w, cfg)
    assert all(np.array_equal(a, b) for a, b in zip(out, imgs))
print("ok", sum(len(c.payload) for c in cs))
