"""Reference values of codec.theoretical_bpsp (codec.py:255-274) for a few
golden images, written to tests/golden/reference_theoretical.json.  Runs the
REFERENCE package read-only in this container (like gen_golden.py):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_theory.py

The images are the golden container images already in reference_vectors.npz.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from lpic import codec  # noqa: E402  (the reference)

from gen_golden import weights_for  # noqa: E402

OUT = os.path.join(HERE, "..", "tests", "golden", "reference_theoretical.json")


def main():
    g = np.load(os.path.join(HERE, "..", "tests", "golden", "reference_vectors.npz"))
    cases = ["small.glorot7.nat13x17.seq", "small.glorot7.nat13x17.wave", "small.glorot7.nat13x17.diag",
             "small.glorot7.rand9x8.seq", "small_logistic.glorot3.nat13x17.seq", "tiny.glorot7.nat13x17.wave",
             "ref.kaiming0.c1.seq", "ref.kaiming0.c1.diag", "h1.glorot5.nat13x17.wave"]
    res = {}
    for cid in cases:
        name, initseed, key, mode = cid.split(".")
        init = "glorot" if initseed.startswith("glorot") else "kaiming"
        w, cfg = weights_for(name, init, int(initseed[len(init):]))
        img = g[f"cont_{cid}_image"]
        res[cid] = float(codec.theoretical_bpsp(img, w, cfg, mode))
        print(cid, res[cid])
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
