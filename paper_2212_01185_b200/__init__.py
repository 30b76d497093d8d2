"""B200-native hot path of the LPPLIC learned lossless codec (arXiv 2212.01185).

Drop-in for the reference package (/root/reference/pkg/src/lpic/__init__.py:11-26):
the same public names for the codec, coder, mixture, network, schedule and
training API, importable as ``lpic`` too (lpic/__init__.py).  Network
evaluation, CDF construction, range coding and the wavefront decoder run in
liblpic_b200.so (sm_100a) with no CPU fallback; the scipy mixture helpers
and the interactive RangeDecoder are host utilities outside the codec path
(mixture.py, coder.py).
"""

from .codec import (CodecTrace, Container, bpsp, decode, decode_batch, encode, encode_batch,
                    theoretical_bpsp)
from .coder import RangeDecoder, RangeEncoder, rate_of
from .mixture import PixelParams, activate, bin_probability, pmf, quantize_cdf, update_means
from .errors import CorruptStreamError, FingerprintMismatchError, LpicError, UnsupportedImageError
from .network import (Distribution, ModelConfig, Weights, causal_taps, count_parameters, estimate_macs,
                      forward_fc, forward_full, forward_patch, forward_taps_batch, glorot_weights,
                      get_precision, kaiming_weights, leaky_relu, load_weights, normalize, normalize_value,
                      save_weights, set_precision, weight_fingerprint, zero_weights)
from .tiles import (TiledContainer, bits_per_gray_pixel, decode_gray, decode_tiled, encode_gray, encode_gray_batch,
                    encode_tiled, gray_to_rgb, tile_grid)
from .schedules import (Schedule, ScheduleMode, build_schedule, diagonal, parse_mode, sequential, validate,
                        wavefront)
from .training import TrainConfig, train

__version__ = "0.1.0"
