"""Generate tests/golden/ fixtures by running the REFERENCE package itself.

Run here (the reference is importable only in this container):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

It imports /root/reference/pkg/src/lpic read-only and records, with fixed
seeds, the reference's own outputs: CDF tables from kernels.channel_cdfs,
raw planes from network.forward_full, range-coder payloads from
coder.RangeEncoder, containers from codec.encode, and weight fingerprints.
The fixtures pin the C oracle (tests/test_oracle_golden.py) and the GPU
path (tests/test_gpu_*.py); the GPU box never needs /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from lpic import codec, kernels, network, synthetic  # noqa: E402  (the reference)
from lpic.coder import RangeEncoder  # noqa: E402
from lpic.mixture import quantize_cdf  # noqa: E402
from lpic.network import Distribution, ModelConfig, glorot_weights  # noqa: E402

from paper_2212_01185_b200 import synth  # noqa: E402  (harness generators, numpy only)
from paper_2212_01185_b200.network import kaiming_weights  # noqa: E402

CFGS = {
    "ref": ModelConfig(),
    "small": ModelConfig(mixtures=3, filters=16, layers=5),
    "tiny": ModelConfig(mixtures=2, filters=8, layers=4),
    "small_logistic": ModelConfig(mixtures=3, filters=16, layers=5, distribution=Distribution.LOGISTIC),
    "h1": ModelConfig(mixtures=3, filters=16, layers=4, kernel_half=1),
}


def weights_for(name: str, init: str, seed: int):
    cfg = CFGS[name]
    if init == "glorot":
        return glorot_weights(cfg, np.random.default_rng(seed)), cfg
    w = kaiming_weights(cfg, np.random.default_rng(seed))
    ref_w = network.zero_weights(cfg)
    for a, b in zip(ref_w.tensors(), w.tensors()):
        a[:] = b
    return ref_w, cfg


def raw_rows(rng, N, K, narrow_frac=0.5):
    M = 12 * K
    raw = rng.normal(0.0, 1.5, (N, M)).astype(np.float32)
    narrow = rng.random(N) < narrow_frac
    rho = np.where(narrow[:, None], rng.uniform(-6.5, -2.0, (N, 3 * K)), rng.uniform(-2.5, 1.5, (N, 3 * K)))
    raw[:, 6 * K:9 * K] = rho.astype(np.float32)
    raw[:, 3 * K:6 * K] = rng.uniform(-1.2, 1.2, (N, 3 * K)).astype(np.float32)
    # a few extreme rows: clamped scales, saturated means, huge logits
    raw[0, 6 * K:9 * K] = -100.0
    raw[1, 6 * K:9 * K] = 100.0
    raw[2, 3 * K:6 * K] = 5.0
    raw[3, :3 * K] = 60.0
    return raw


def gen_cdfs(out: dict) -> None:
    rng = np.random.default_rng(20240601)
    for tag, K, dist in (("g3", 3, 0), ("g2", 2, 0), ("l3", 3, 1), ("g1", 1, 0)):
        N = 256
        raw = raw_rows(rng, N, K)
        rn = np.array([network.normalize_value(int(v)) for v in rng.integers(0, 256, N)], np.float32)
        gn = np.array([network.normalize_value(int(v)) for v in rng.integers(0, 256, N)], np.float32)
        masses = np.empty((N, 3, 256), np.uint16)
        for ch in range(3):
            t = np.empty((N, 257), np.int64)
            kernels.channel_cdfs(raw, K, dist, ch, rn, gn, kernels.EDGES, t)
            assert t[:, 0].max() == 0 and (t[:, 256] == 65536).all()
            masses[:, ch] = np.diff(t, axis=1).astype(np.uint16)   # mass <= 65281 fits u16
        out[f"cdf_{tag}_raw"] = raw
        out[f"cdf_{tag}_rn"] = rn
        out[f"cdf_{tag}_gn"] = gn
        out[f"cdf_{tag}_masses"] = masses
        out[f"cdf_{tag}_K"] = np.int64(K)
        out[f"cdf_{tag}_dist"] = np.int64(dist)


def gen_quantize(out: dict) -> None:
    rng = np.random.default_rng(77)
    pmfs = []
    for _ in range(64):
        p = rng.dirichlet(np.full(256, float(rng.uniform(0.02, 5.0))))
        pmfs.append(p)
    p = np.zeros(256); p[0] = 1.0; pmfs.append(p)
    pmfs.append(np.full(256, 1.0 / 256.0))
    p = np.zeros(256); p[17] = 0.5; p[200] = 0.5; pmfs.append(p)
    pmfs = np.array(pmfs)
    out["quant_pmf"] = pmfs
    out["quant_cdf"] = np.array([quantize_cdf(p) for p in pmfs], np.int64)


def gen_coder(out: dict) -> None:
    rng = np.random.default_rng(3)
    tables = []
    for _ in range(8):
        tables.append(quantize_cdf(rng.dirichlet(np.full(256, float(rng.uniform(0.02, 5.0))))))
    tables = np.array(tables, np.int64)
    n = 20000
    picks = rng.integers(0, len(tables), n)
    syms = []
    for k in picks:
        masses = np.diff(tables[k]).astype(np.float64)
        syms.append(int(rng.choice(256, p=masses / masses.sum())))
    syms = np.array(syms, np.int64)
    enc = RangeEncoder()
    for s, k in zip(syms, picks):
        enc.encode(int(s), tables[k])
    out["coder_tables"] = tables
    out["coder_picks"] = picks.astype(np.int64)
    out["coder_syms"] = syms
    out["coder_payload"] = np.frombuffer(enc.finish(), np.uint8)
    # uniform and spiked KATs (tests/test_coder.py:39-60)
    uni = np.arange(257, dtype=np.int64) * 256
    s2 = rng.integers(0, 256, 1000)
    enc = RangeEncoder()
    for s in s2:
        enc.encode(int(s), uni)
    out["coder_uniform_syms"] = s2.astype(np.int64)
    out["coder_uniform_payload"] = np.frombuffer(enc.finish(), np.uint8)


def gen_network(out: dict, meta: dict) -> None:
    for name, init, seed in (("small", "glorot", 7), ("ref", "kaiming", 0), ("tiny", "glorot", 7), ("h1", "glorot", 5)):
        w, cfg = weights_for(name, init, seed)
        img = synthetic.natural_like(np.random.default_rng(11), 16, 16)
        raw = network.forward_full(network.normalize(img), w, cfg)
        out[f"net_{name}_image"] = img
        out[f"net_{name}_raw"] = raw
        meta[f"fingerprint_{name}_{init}{seed}"] = int(network.weight_fingerprint(w, cfg))


def gen_containers(out: dict, meta: dict) -> None:
    cases = []
    rng = np.random.default_rng(5)
    imgs = {
        "rand9x8": rng.integers(0, 256, (9, 8, 3), dtype=np.uint8),
        "nat13x17": synthetic.natural_like(rng, 13, 17),
        "one": np.array([[[13, 200, 77]]], np.uint8),
        "row1x7": rng.integers(0, 256, (1, 7, 3), dtype=np.uint8),
        "col6x1": rng.integers(0, 256, (6, 1, 3), dtype=np.uint8),
    }
    for pname, pimg in synthetic.pathological_images(12).items():
        imgs["path_" + pname] = pimg
    plan = [("small", "glorot", 7, list(imgs)), ("tiny", "glorot", 7, ["rand9x8", "nat13x17", "one"]),
            ("small_logistic", "glorot", 3, ["rand9x8", "nat13x17"]), ("h1", "glorot", 5, ["rand9x8", "nat13x17"]),
            ("ref", "kaiming", 0, ["nat13x17", "rand9x8"])]
    for name, init, seed, keys in plan:
        w, cfg = weights_for(name, init, seed)
        for key in keys:
            for mode in ("seq", "wave", "diag"):
                if mode == "diag" and cfg.kernel_half != 2:
                    continue
                c = codec.encode(imgs[key], w, cfg, mode)
                cid = f"{name}.{init}{seed}.{key}.{mode}"
                cases.append(cid)
                out[f"cont_{cid}_image"] = imgs[key]
                out[f"cont_{cid}_bytes"] = np.frombuffer(c.to_bytes(), np.uint8)
    # BASELINE configs[0]: C1 1/f 64x64, Kaiming seed 0, all modes
    w, cfg = weights_for("ref", "kaiming", 0)
    img = synth.c1_image()
    for mode in ("seq", "wave", "diag"):
        c = codec.encode(img, w, cfg, mode)
        cid = f"ref.kaiming0.c1.{mode}"
        cases.append(cid)
        out[f"cont_{cid}_image"] = img
        out[f"cont_{cid}_bytes"] = np.frombuffer(c.to_bytes(), np.uint8)
        meta[f"bpsp_{cid}"] = codec.bpsp(c)
    meta["container_cases"] = cases


def gen_large(meta: dict) -> None:
    """One C2-geometry image (768x512): the reference payload's length and
    sha256 (the bytes themselves are regenerated by the C oracle)."""
    w, cfg = weights_for("ref", "kaiming", 0)
    img = synth.synth_1f(0, 512, 768)
    meta["c2_image_sha256"] = hashlib.sha256(img.tobytes()).hexdigest()
    c = codec.encode(img, w, cfg, "wave")
    meta["c2_seed0_wave_len"] = len(c.payload)
    meta["c2_seed0_wave_sha256"] = hashlib.sha256(c.payload).hexdigest()
    meta["c2_seed0_wave_bpsp"] = codec.bpsp(c)


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    out: dict = {}
    meta: dict = {"generator": "oracle/gen_golden.py", "reference": "/root/reference/pkg/src/lpic (lpic 0.1.0)"}
    gen_cdfs(out)
    gen_quantize(out)
    gen_coder(out)
    gen_network(out, meta)
    gen_containers(out, meta)
    meta["c1_image_sha256"] = hashlib.sha256(synth.c1_image().tobytes()).hexdigest()
    if "--no-large" not in sys.argv:
        gen_large(meta)
    np.savez_compressed(os.path.join(OUT, "reference_vectors.npz"), **out)
    with open(os.path.join(OUT, "reference_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays;", os.path.getsize(os.path.join(OUT, "reference_vectors.npz")), "bytes")


if __name__ == "__main__":
    main()
