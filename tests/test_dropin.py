"""The drop-in modules beside the codec -- synthetic, mixture, images, cli,
the host RangeDecoder and the ``lpic`` import alias -- against fixtures that
oracle/gen_golden_dropin.py wrote by running the reference itself
(tests/golden/reference_dropin.npz).  CPU only (the GPU halves -- the
RangeEncoder and the kernels seam -- are in test_gpu_parity.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def G():
    return dict(np.load(os.path.join(GOLDEN, "reference_dropin.npz")))


def test_lpic_alias_resolves_to_this_package():
    import lpic
    import lpic.codec
    import lpic.kernels
    import paper_2212_01185_b200 as P
    assert lpic.codec is P.codec and lpic.kernels is P.kernels
    for name in ("encode", "decode", "Container", "RangeEncoder", "RangeDecoder", "rate_of", "activate", "pmf",
                 "quantize_cdf", "update_means", "bin_probability", "PixelParams", "TrainConfig", "train",
                 "ModelConfig", "Weights", "wavefront", "validate"):
        assert getattr(lpic, name) is getattr(P, name)
    from lpic.schedules import DIAGONAL_UNAVAILABLE  # noqa: F401
    from lpic.images import load_image  # noqa: F401
    from lpic.cli import main  # noqa: F401


def test_synthetic_matches_reference(G):
    from paper_2212_01185_b200 import synthetic as S
    for s in range(3):
        assert np.array_equal(S.natural_like(np.random.default_rng(s), 17 + s, 23 - s), G[f"natural_{s}"])
        assert np.array_equal(S.causal_mean_image(np.random.default_rng(100 + s), 13, 11 + s), G[f"causal_{s}"])
    for name, im in S.pathological_images(12).items():
        assert np.array_equal(im, G[f"path_{name}"])
    assert S.conditional_entropy_bits(list(G["centropy_corpus"])) == float(G["centropy_bits"])


def test_mixture_matches_reference(G):
    from paper_2212_01185_b200 import mixture as Mx
    from paper_2212_01185_b200.network import Distribution, ModelConfig
    for K, dist in ((3, 0), (2, 1)):
        cfg = ModelConfig(mixtures=K, filters=8, layers=3, distribution=Distribution(dist))
        raws = G[f"mix{K}{dist}_raw"]
        pm, cd, mu = [], [], []
        for raw in raws:
            q = Mx.update_means(Mx.activate(raw, cfg), 0.25, -0.5)
            mu.append(q.means)
            for ch in range(3):
                v = Mx.pmf(q, ch, cfg.distribution)
                pm.append(v)
                cd.append(Mx.quantize_cdf(v))
        assert np.array_equal(np.stack(mu), G[f"mix{K}{dist}_means"])
        assert np.array_equal(np.stack(pm), G[f"mix{K}{dist}_pmf"])
        assert np.array_equal(np.stack(cd), G[f"mix{K}{dist}_cdf"])
    got = [Mx.bin_probability(x, 0.1, 0.3, d) for d in (0, 1) for x in (0, 17, 128, 255)]
    assert np.array_equal(np.array(got), G["binprob"])
    with pytest.raises(ValueError):
        Mx.activate(np.zeros(5, np.float32), ModelConfig())
    with pytest.raises(ValueError):
        Mx.quantize_cdf(np.full(256, np.nan))


def test_host_range_decoder_reads_reference_stream(G):
    """The reference RangeEncoder's bytes decode to the same symbols with the
    host RangeDecoder; a truncated stream raises CorruptStreamError."""
    from paper_2212_01185_b200.coder import RangeDecoder
    from paper_2212_01185_b200.errors import CorruptStreamError
    tabs, picks, syms, pay = G["rc_tables"], G["rc_picks"], G["rc_syms"], G["rc_payload"].tobytes()
    d = RangeDecoder(pay)
    assert [d.decode(tabs[t]) for t in picks] == [int(s) for s in syms]
    d = RangeDecoder(pay[:len(pay) // 2])
    with pytest.raises(CorruptStreamError):
        for t in picks:
            d.decode(tabs[t])
    RangeDecoder(bytes(3))                                  # a flush-only stream constructs


def test_images_ppm_png(G, tmp_path):
    from paper_2212_01185_b200 import images
    from paper_2212_01185_b200.errors import UnsupportedImageError
    img = G["natural_0"]
    p = tmp_path / "x.ppm"
    images.save_image(p, img)
    assert p.read_bytes() == G["ppm_bytes"].tobytes()
    assert np.array_equal(images.load_image(p), img)
    q = tmp_path / "x.png"
    images.save_image(q, img)
    assert np.array_equal(images.load_image(q), img)
    c = tmp_path / "c.ppm"
    c.write_bytes(b"P6\n# comment\n1 1\n# more\n255\n\x01\x02\x03")
    assert images.load_image(c)[0, 0].tolist() == [1, 2, 3]
    for data, msg in ((b"P6\n1 1\n65535\n\0\0\0\0\0\0", "maxval"), (b"P6\n4 4\n255\n\0\0", "truncated"),
                      (b"P5\n1 1\n255\n\0", "P6")):
        bad = tmp_path / "bad.ppm"
        bad.write_bytes(data)
        with pytest.raises(UnsupportedImageError, match=msg):
            images.load_image(bad)
    empty = tmp_path / "nothing"
    empty.mkdir()
    with pytest.raises(UnsupportedImageError):
        images.load_corpus(empty)


def test_cli_parser_surface():
    from paper_2212_01185_b200 import cli
    ap = cli.build_parser()
    a = ap.parse_args(["encode", "-i", "a.ppm", "-w", "m.lpwt", "-m", "wave", "-o", "a.lpic"])
    assert (a.command, a.mode) == ("encode", "wave")
    a = ap.parse_args(["bench", "-d", "dir", "-w", "m.lpwt", "--csv", "r.csv"])
    assert a.mode == "seq"
    with pytest.raises(SystemExit):
        ap.parse_args(["encode", "-i", "x", "-w", "y", "--bogus", "z"])
    assert cli._grid("K=3,5;C=8;dist=gaussian,logistic")[1] == {"K": 3, "C": 8, "L": 5, "dist": "logistic"}
    with pytest.raises(ValueError):
        cli._grid("Q=1")
