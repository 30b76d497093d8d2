import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(GOLDEN, "reference_vectors.npz")))


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "reference_meta.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle


CFG_ARGS = {
    "ref": dict(),
    "small": dict(mixtures=3, filters=16, layers=5),
    "tiny": dict(mixtures=2, filters=8, layers=4),
    "small_logistic": dict(mixtures=3, filters=16, layers=5, distribution=1),
    "h1": dict(mixtures=3, filters=16, layers=4, kernel_half=1),
}


def make_weights(name: str, init: str, seed: int):
    from paper_2212_01185_b200.network import Distribution, ModelConfig, glorot_weights, kaiming_weights
    args = dict(CFG_ARGS[name])
    if "distribution" in args:
        args["distribution"] = Distribution(args["distribution"])
    cfg = ModelConfig(**args)
    rng = np.random.default_rng(seed)
    w = glorot_weights(cfg, rng) if init == "glorot" else kaiming_weights(cfg, rng)
    return w, cfg


def parse_case(cid: str):
    name, initseed, key, mode = cid.split(".")
    init = "glorot" if initseed.startswith("glorot") else "kaiming"
    seed = int(initseed[len(init):])
    return name, init, seed, key, mode


def oracle_weights(oracle, w, cfg):
    return oracle.OracleWeights(w.tensors(), cfg.mixtures, cfg.filters, cfg.layers, cfg.kernel_half,
                                int(cfg.distribution))
