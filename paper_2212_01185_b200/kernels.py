"""The kernel seam (drop-in for /root/reference/pkg/src/lpic/kernels.py).

The reference's numba kernels take plain arrays and write into an
out-parameter.  Here every one of them runs on the B200 through
liblpic_b200.so with the same signature, so callers of the seam see the
same results (bit-identical network outputs and tables, tests/golden):

  forward_full_f32 / forward_taps_f32 / forward_fc_f32  -> lpic_forward_full / lpic_forward_taps
  channel_cdfs       -> lpic_channel_cdfs      (kernels.py:296-313)
  true_symbol_probs  -> lpic_true_symbol_probs (kernels.py:316-346)
  _quantized_cdf     -> lpic_quantized_cdf     (kernels.py:250-293)

``reference_forward_full`` stays what it is in the reference: the plain
numpy statement of the canonical float32 accumulation order that the
compiled paths are pinned against (test infrastructure, not a fallback).
"""

from __future__ import annotations

import numpy as np

from . import _native, network
from .network import Distribution, ModelConfig, Weights

LEAKY_SLOPE = np.float32(0.01)
EDGES = (2.0 * np.arange(257, dtype=np.float64) - 256.0) / 255.0
CDF_TOTAL = 65536
CDF_FLOOR_TOTAL = CDF_TOTAL - 256


def causal_tap_offsets(kernel_half: int) -> np.ndarray:
    """Canonical causal tap order: the h rows above (dj = -h..h), then the h
    positions left of the centre; (T, 2) int64."""
    return network.causal_taps(kernel_half)


def _model_of(masked_w, masked_b, hidden_w, hidden_b, out_w, out_b):
    T, _, Cf = masked_w.shape
    h = next((k for k in range(1, 64) if (2 * k + 1) * k + k == T), None)
    if h is None:
        raise ValueError(f"tap count {T} is not a causal kernel")
    M = out_w.shape[0]
    if M % 12:
        raise ValueError("output width must be 12 * mixtures")
    cfg = ModelConfig(mixtures=M // 12, filters=Cf, layers=hidden_w.shape[0] + 2, kernel_half=h,
                      distribution=Distribution.GAUSSIAN)
    w = Weights(*(np.ascontiguousarray(a, np.float32) for a in (masked_w, masked_b, hidden_w, hidden_b, out_w, out_b)))
    return w, cfg


def forward_full_f32(x, taps, masked_w, masked_b, hidden_w, hidden_b, out_w, out_b, out):
    """(H, W, 3) f32 -> out (H, W, M) f32, canonical order."""
    w, cfg = _model_of(masked_w, masked_b, hidden_w, hidden_b, out_w, out_b)
    if not np.array_equal(np.asarray(taps), network.causal_taps(cfg.kernel_half)):
        raise ValueError("only the canonical causal tap order is supported")
    out[...] = network.forward_full(np.ascontiguousarray(x, np.float32), w, cfg)


def forward_taps_f32(tap_x, masked_w, masked_b, hidden_w, hidden_b, out_w, out_b, out):
    """(N, T, 3) gathered taps -> out (N, M)."""
    w, cfg = _model_of(masked_w, masked_b, hidden_w, hidden_b, out_w, out_b)
    out[...] = network.forward_taps_batch(np.ascontiguousarray(tap_x, np.float32), w, cfg)


def forward_fc_f32(ctx, masked_w, masked_b, hidden_w, hidden_b, out_w, out_b, out):
    """(N, 3T) flattened context (tap-major, channel-minor) -> out (N, M)."""
    w, cfg = _model_of(masked_w, masked_b, hidden_w, hidden_b, out_w, out_b)
    c = np.ascontiguousarray(ctx, np.float32)
    out[...] = network.forward_taps_batch(c.reshape(c.shape[0], cfg.tap_count, 3), w, cfg)


def reference_forward_full(x, taps, masked_w, masked_b, hidden_w, hidden_b, out_w, out_b):
    """numpy statement of the canonical float32 order (the parity oracle of
    the compiled paths): taps ascending, input channels ascending, dense
    inputs ascending, every product rounded then added, bias last."""
    H, W, _ = x.shape
    acc = np.zeros((H, W, masked_b.shape[0]), np.float32)
    for t, (di, dj) in enumerate(np.asarray(taps, dtype=np.int64)):
        src = np.zeros((H, W, 3), np.float32)
        ys, xs = slice(max(0, -di), min(H, H - di)), slice(max(0, -dj), min(W, W - dj))
        if ys.start < ys.stop and xs.start < xs.stop:
            src[ys, xs] = x[ys.start + di:ys.stop + di, xs.start + dj:xs.stop + dj]
        for c in range(3):
            acc = acc + src[:, :, c:c + 1] * masked_w[t, c, :]
    acc = acc + masked_b
    a = np.where(acc >= 0, acc, LEAKY_SLOPE * acc)
    for l in range(hidden_w.shape[0]):
        acc = np.zeros_like(a)
        for i in range(a.shape[2]):
            acc = acc + a[:, :, i:i + 1] * hidden_w[l, :, i]
        acc = acc + hidden_b[l]
        a = np.where(acc >= 0, acc, LEAKY_SLOPE * acc)
    raw = np.zeros((H, W, out_b.shape[0]), np.float32)
    for i in range(a.shape[2]):
        raw = raw + a[:, :, i:i + 1] * out_w[:, i]
    return raw + out_b


def _dev(a, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype)).cuda()


def channel_cdfs(raw, K, dist, channel, rn, gn, edges, out):
    """raw (N, M) f32, rn/gn (N,) f32 -> out (N, 257) int64 quantised tables
    of one channel (the cross-channel mean update folded in)."""
    import torch
    L = _native.require_cuda()
    raw = np.ascontiguousarray(raw, np.float32)
    N, M = raw.shape
    if N == 0:
        return
    d_out = torch.empty((N, 257), dtype=torch.int32, device="cuda")
    # (device copies held in locals: a temporary's memory could be recycled
    # by the caching allocator before the kernel reads it)
    d_raw, d_rn, d_gn = _dev(raw, np.float32), _dev(rn, np.float32), _dev(gn, np.float32)
    _native.check(L.lpic_channel_cdfs(d_raw.data_ptr(), N, M, int(K), int(dist), int(channel), d_rn.data_ptr(),
                                      d_gn.data_ptr(), d_out.data_ptr(), _native.stream_ptr()), "lpic_channel_cdfs")
    out[...] = d_out.cpu().numpy()


def true_symbol_probs(raw, syms, rn, gn, K, dist, edges, out):
    """Unquantised probability of each coded sub-pixel -> out (N, 3) f64."""
    from .codec import true_symbol_probs as tsp
    out[...] = tsp(raw, syms, rn, gn, int(K), int(dist))


def _quantized_cdf(pi, mu, s, K, dist, edges, cdf, pmf=None, neg_rem=None):
    """One table from explicit mixture parameters (pi, mu, s: (K,) f64) ->
    cdf (257,) int64; like the reference kernel it also leaves the PMF in
    `pmf` and floor - value in `neg_rem` (256 each) when they are given."""
    import torch
    L = _native.require_cuda()
    d_out = torch.empty((1, 257), dtype=torch.int32, device="cuda")
    d_pmf = torch.empty((1, 256), dtype=torch.float64, device="cuda")
    d_neg = torch.empty((1, 256), dtype=torch.float64, device="cuda")
    d_pi, d_mu, d_s = (_dev(np.asarray(a)[:K], np.float64) for a in (pi, mu, s))
    _native.check(L.lpic_quantized_cdf(d_pi.data_ptr(), d_mu.data_ptr(), d_s.data_ptr(), 1, int(K), int(dist),
                                       d_out.data_ptr(), d_pmf.data_ptr() if pmf is not None else None,
                                       d_neg.data_ptr() if neg_rem is not None else None, _native.stream_ptr()),
                  "lpic_quantized_cdf")
    cdf[...] = d_out.cpu().numpy()[0]
    if pmf is not None:
        pmf[...] = d_pmf.cpu().numpy()[0]
    if neg_rem is not None:
        neg_rem[...] = d_neg.cpu().numpy()[0]
