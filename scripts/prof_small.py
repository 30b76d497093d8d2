"""Small fixed workload for ncu: encode + decode a few 1/f images once."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import synth

H = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w, cfg = synth.baseline_weights()
imgs = synth.batch(n, H, H)
cs = P.encode_batch(imgs, w, cfg, "wave")
outs = P.decode_batch(cs, w, cfg)
assert all(np.array_equal(a, b) for a, b in zip(outs, imgs))
print("ok", sum(len(c.payload) for c in cs))
