"""CPU tests of the host-side mirror of the reference API (no GPU calls):
schedules, configs, weights/LPWT/fingerprint, containers, synthetic inputs.
Expected values are the reference's own known answers
(/root/reference/pkg/tests/test_schedules.py, test_network.py, test_codec.py)."""

import hashlib

import numpy as np
import pytest

from conftest import make_weights
import paper_2212_01185_b200 as P
from paper_2212_01185_b200 import codec, network, schedules, synth


def test_sequential_counts():
    assert P.sequential(2, 2).step_count == 4
    s = P.sequential(1, 5)
    assert [st[0] for st in s.steps] == [(0, j) for j in range(5)]
    for d in (3, 16, 64):
        assert P.sequential(d, d).step_count == d * d


def test_wavefront_step_formula():
    assert P.wavefront(512, 512, 2).step_count == 2045
    assert P.wavefront(4, 4, 2).step_count == 13
    for d in range(1, 40):
        assert P.wavefront(d, d, 2).step_count == d + (d - 1) * 3
    for h in (1, 2, 3):
        for d in (1, 2, 7, 16):
            assert P.wavefront(d, d, h).step_count == d + (d - 1) * (h + 1)


def test_wavefront_assignment_and_geometry():
    s = P.wavefront(5, 5, 2)
    step_of = {p: t for t, st in enumerate(s.steps) for p in st}
    assert step_of[(1, 0)] == 3 and step_of[(0, 3)] == 3
    assert all(t == 3 * i + j for (i, j), t in step_of.items())
    # SURVEY Appendix B.6 geometry table
    for (W, H), steps, maxpx in [((64, 64), 253, 22), ((768, 512), 2301, 256), ((2048, 1536), 6653, 683),
                                 ((512, 512), 2045, 171), ((256, 256), 1021, 86)]:
        assert schedules.step_count("wave", H, W, 2) == steps
        a = 3
        widest = max(min(H - 1, t // a) - max(0, -(-(t - W + 1) // a)) + 1 for t in range(steps))
        assert widest == maxpx


def test_diagonal_counts_and_substitutions():
    assert P.diagonal(512, 512, 2).step_count == 1023
    for d in range(1, 30):
        assert P.diagonal(d, d, 2).step_count == 2 * d - 1
    with pytest.raises(ValueError):
        P.diagonal(4, 4, 1)
    s = P.diagonal(12, 12, 2)
    for off in schedules.DIAGONAL_UNAVAILABLE:
        assert s.substitutions[(5, 5, *off)] == (3, 6)
    assert P.validate(s, 2) == []


@pytest.mark.parametrize("mode", ["seq", "wave", "diag"])
def test_validate_exhaustive(mode):
    for H, W in [(1, 1), (1, 7), (6, 1), (5, 9), (9, 5), (8, 8)]:
        assert P.validate(P.build_schedule(mode, H, W, 2), 2) == []


def test_coding_order_matches_schedule_and_oracle(oracle_mod):
    for mode in ("seq", "wave", "diag"):
        for H, W in [(1, 1), (3, 11), (9, 8), (13, 17)]:
            order = codec.coding_order(mode, H, W, 2)
            flat = [p for st in P.build_schedule(mode, H, W, 2).steps for p in st]
            assert [tuple(p) for p in order] == flat
            o, passes = oracle_mod.coding_order(mode, H, W, 2)
            assert np.array_equal(o, order)
            assert passes == schedules.nonempty_step_count(mode, H, W, 2)


def test_pass_counts_8x8():
    # tests/test_codec.py:162-170 of the reference
    assert schedules.nonempty_step_count("seq", 8, 8, 2) == 64
    assert schedules.nonempty_step_count("wave", 8, 8, 2) == 29
    assert schedules.nonempty_step_count("diag", 8, 8, 2) == 15


def test_parse_mode():
    assert P.parse_mode("wave") == P.ScheduleMode.WAVEFRONT
    assert P.parse_mode("DIAGONAL") == P.ScheduleMode.DIAGONAL
    with pytest.raises(ValueError):
        P.parse_mode("zigzag")


@pytest.mark.parametrize("kw,expected", [
    (dict(), 58916), (dict(mixtures=5), 62012), (dict(mixtures=7), 65108), (dict(filters=64), 17188),
    (dict(filters=192), 125220), (dict(layers=4), 42404), (dict(layers=6), 75428)])
def test_count_parameters(kw, expected):
    cfg = P.ModelConfig(**kw)
    assert P.count_parameters(cfg) == expected
    assert sum(t.size for t in P.zero_weights(cfg).tensors()) == expected


def test_macs_and_config():
    cfg = P.ModelConfig()
    assert P.estimate_macs(cfg, 1, 1) == 58368
    assert P.estimate_macs(cfg, 512, 512) == 15_300_820_992
    assert cfg.param_channels == 36
    with pytest.raises(ValueError):
        P.ModelConfig(mixtures=0)
    with pytest.raises(ValueError):
        P.ModelConfig(layers=2)


def test_causal_taps_reference_kernel():
    assert [tuple(t) for t in P.causal_taps(2)] == [(-2, -2), (-2, -1), (-2, 0), (-2, 1), (-2, 2), (-1, -2),
                                                   (-1, -1), (-1, 0), (-1, 1), (-1, 2), (0, -2), (0, -1)]


def test_normalize(oracle_mod):
    img = np.arange(256, dtype=np.uint8).reshape(16, 16)
    xn = P.normalize(np.stack([img] * 3, axis=2))
    assert xn[0, 0, 0] == -1.0 and xn[15, 15, 0] == 1.0 and xn.dtype == np.float32
    for v in range(256):
        assert P.normalize_value(v) == xn[v // 16, v % 16, 0] == np.float32(oracle_mod.normalize_value(v))


def test_fnv_vectors_native():
    assert network.fnv1a64(b"") == 0xcbf29ce484222325
    assert network.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    assert network.fnv1a64(b"foobar") == 0x85944171f73967e8


def test_weight_init_matches_reference_fingerprints(golden_meta):
    for name, init, seed in (("small", "glorot", 7), ("ref", "kaiming", 0), ("tiny", "glorot", 7), ("h1", "glorot", 5)):
        w, cfg = make_weights(name, init, seed)
        assert P.weight_fingerprint(w, cfg) == golden_meta[f"fingerprint_{name}_{init}{seed}"]


def test_weight_file_roundtrip_and_flip(tmp_path):
    w, cfg = make_weights("small", "glorot", 7)
    path = tmp_path / "m.lpwt"
    fp = P.save_weights(path, w, cfg)
    w2, cfg2 = P.load_weights(path)
    assert cfg2 == cfg and fp == P.weight_fingerprint(w2, cfg2)
    for a, b in zip(w.tensors(), w2.tensors()):
        assert np.array_equal(a, b)
    blob = bytearray(path.read_bytes())
    blob[len(blob) // 2] ^= 1
    path.write_bytes(bytes(blob))
    with pytest.raises(P.LpicError, match="fingerprint"):
        P.load_weights(path)


def test_check_weights_errors():
    w, cfg = make_weights("small", "glorot", 7)
    bad = w.copy()
    bad.out_b = bad.out_b[:-1]
    with pytest.raises(P.LpicError):
        network.check_weights(bad, cfg)
    bad = w.copy()
    bad.masked_b = bad.masked_b.astype(np.float64)
    with pytest.raises(P.LpicError):
        network.check_weights(bad, cfg)


def test_container_roundtrip(golden, golden_meta):
    for cid in golden_meta["container_cases"][:10]:
        blob = golden[f"cont_{cid}_bytes"].tobytes()
        c = P.Container.from_bytes(blob)
        assert c.to_bytes() == blob
    with pytest.raises(P.LpicError):
        P.Container.from_bytes(b"JUNK" + blob[4:])
    with pytest.raises(P.LpicError):
        P.Container.from_bytes(blob[:-1])
    c = P.Container(P.ScheduleMode.SEQUENTIAL, 3, 0, 16, 16, 0, b"x" * 100)
    assert P.bpsp(c) == pytest.approx(800.0 / 768.0)


def test_input_validation_before_gpu():
    w, cfg = make_weights("small", "glorot", 7)
    with pytest.raises(ValueError):
        P.encode(np.zeros((4, 4), np.uint8), w, cfg, "seq")
    with pytest.raises(ValueError):
        P.encode(np.zeros((4, 4, 3), np.float32), w, cfg, "seq")
    with pytest.raises(ValueError):
        P.encode(np.zeros((4, 4, 3), np.uint8), w, cfg, "zigzag")


def test_synthetic_generators(golden_meta):
    img = synth.c1_image()
    assert img.shape == (64, 64, 3) and img.dtype == np.uint8
    assert hashlib.sha256(img.tobytes()).hexdigest() == golden_meta["c1_image_sha256"]
    b = synth.batch(3, 32, 48)
    assert b.shape == (3, 32, 48, 3)
    corr = np.corrcoef(b[0, ..., 0].ravel().astype(float), b[0, ..., 1].ravel().astype(float))[0, 1]
    assert corr > 0.5


def test_tile_grid_and_container_roundtrip():
    from paper_2212_01185_b200 import tiles
    g = tiles.tile_grid(1100, 700, 512, 512)
    assert len(g) == 6 and g[-1] == (1024, 512, 76, 188)
    assert sum(h * w for _, _, h, w in g) == 1100 * 700
    conts = [P.Container(P.ScheduleMode.WAVEFRONT, 3, 0, w, h, 0x1234, bytes([k]) * (k + 3))
             for k, (_, _, h, w) in enumerate(g)]
    tc = tiles.TiledContainer(1100, 700, 512, 512, conts)
    back = tiles.TiledContainer.from_bytes(tc.to_bytes())
    assert (back.height, back.width, back.tile_h, back.tile_w) == (1100, 700, 512, 512)
    assert [c.to_bytes() for c in back.tiles] == [c.to_bytes() for c in conts]
    with pytest.raises(P.LpicError):
        tiles.TiledContainer.from_bytes(tc.to_bytes()[:-1])
    with pytest.raises(P.LpicError):
        tiles.TiledContainer.from_bytes(b"XXXX" + tc.to_bytes()[4:])


def test_gray_helpers():
    g = synth.synth_1f_gray(3, 16, 20)
    assert g.shape == (16, 20) and g.dtype == np.uint8
    rgb = P.gray_to_rgb(g)
    assert rgb.shape == (16, 20, 3) and np.array_equal(rgb[:, :, 1], g)
    with pytest.raises(ValueError):
        P.gray_to_rgb(rgb)


def test_training_api_mirrors_reference():
    """The GPU trainer exposes the reference trainer's names and config
    fields (training.py:34-60, 219-333) and refuses to run without CUDA."""
    import dataclasses
    from paper_2212_01185_b200 import training
    for name in ("TrainConfig", "GradientSet", "zero_gradients", "learning_rate", "loss", "backward", "Adam",
                 "EpochStats", "train", "write_curve"):
        assert hasattr(training, name), name
    fields = [f.name for f in dataclasses.fields(training.TrainConfig)]
    assert fields == ["batch_size", "crop", "lr", "lr_decay", "lr_decay_every", "epochs", "seed", "beta1", "beta2",
                      "eps"]
    tc = training.TrainConfig(lr=1e-3, lr_decay=0.5, lr_decay_every=2)
    assert training.learning_rate(tc, 0) == 1e-3 and training.learning_rate(tc, 5) == 1e-3 * 0.25
    with pytest.raises(ValueError):
        training.TrainConfig(lr=0.0)


def _f32_round(x):
    """Exact round-to-nearest-even of a Fraction to an IEEE float32 value."""
    import math
    from fractions import Fraction as F
    if x == 0:
        return F(0)
    s, x = (-1 if x < 0 else 1), abs(x)
    e = math.floor(math.log2(x.numerator) - math.log2(x.denominator))
    while F(2) ** e > x:
        e -= 1
    while F(2) ** (e + 1) <= x:
        e += 1
    q = x / F(2) ** (e - 23)
    n = q.numerator // q.denominator
    rem = q - n
    if rem > F(1, 2) or (rem == F(1, 2) and n % 2 == 1):
        n += 1
    return s * n * F(2) ** (e - 23)


def test_gather_normalisation_fma_equals_division():
    """csrc/lpic_sched.cuh NormU8: v * rcp with one FMA residual correction is
    the correctly rounded v / 127.5 for every byte (so the FAST encoder's
    in-register normalisation equals the __fdiv_rn tables, network.py:172-177)."""
    from fractions import Fraction as F
    rcp = _f32_round(F(2, 255))
    for v in range(256):
        q0 = _f32_round(F(v) * rcp)
        q = _f32_round(_f32_round(-q0 * F(255, 2) + F(v)) * rcp + q0)
        assert q == _f32_round(F(v) / F(255, 2)), v
