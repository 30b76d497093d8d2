"""C2 encode in FAST precision once (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
w, cfg = synth.baseline_weights()
imgs = synth.batch(n, 512, 768)
P.set_precision("fast")
cs = P.encode_batch(imgs, w, cfg, "wave")
print("ok", sum(len(c.payload) for c in cs))
