"""The public range-coder API (drop-in for /root/reference/pkg/src/lpic/coder.py).

Same bitstream as the codec's device coder: a 48-bit range, 16-bit tables,
renormalisation by whole bytes below 2^40, carries rippling into the
emitted bytes, a 3-byte flush, and a 6-byte decoder window that may read at
most 3 virtual zero bytes past the end (coder.py:1-14, 30-112).

* ``RangeEncoder`` collects (start, width) per ``encode`` call and codes
  the whole stream on the GPU at ``finish()`` with the codec's parallel
  coder (``lpic_rc_encode_streams``: plan, per-chunk coding, carry merge --
  byte-identical to the sequential coder).
* ``RangeDecoder`` returns one symbol per ``decode(cdf)`` and the caller
  chooses the next table from it, so it runs as host code in the same
  library (``lpic_rc_dec_*``; a device round trip per symbol would cost far
  more than the symbol).  The codec's own decoding runs on the GPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .errors import CorruptStreamError

RANGE_BITS = 48
TOTAL_BITS = 16
FLUSH_BYTES = 3
WINDOW_BYTES = RANGE_BITS // 8


class RangeEncoder:
    def __init__(self):
        self._sw: list = []          # start << 16 | (width - 1), the device coder's symbol word
        self._finished = False

    def encode(self, symbol: int, cdf) -> None:
        """Narrow the interval to [cdf[symbol], cdf[symbol+1]) / 65536."""
        if self._finished:
            raise RuntimeError("encoder already finished")
        start = int(cdf[symbol])
        width = int(cdf[symbol + 1]) - start
        if not (0 <= start < 65536 and 1 <= width <= 65536 - start):
            raise ValueError("symbol outside a valid 16-bit cumulative table")
        self._sw.append((start << 16) | (width - 1))

    def finish(self) -> bytes:
        """Code the collected symbols on the GPU and flush; afterwards the
        encoder must not be reused."""
        import torch
        if self._finished:
            raise RuntimeError("encoder already finished")
        self._finished = True
        L = _native.require_cuda()
        n = len(self._sw)
        cap = 6 * n + 64
        d_sw = torch.tensor(np.asarray(self._sw, np.uint32).view(np.int32) if n else np.zeros(1, np.int32),
                            device="cuda")
        d_off = torch.zeros(1, dtype=torch.int64, device="cuda")
        d_cnt = torch.full((1,), n, dtype=torch.int64, device="cuda")
        d_out = torch.zeros(cap, dtype=torch.uint8, device="cuda")
        d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
        d_st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _native.check(L.lpic_rc_encode_streams(d_sw.data_ptr(), d_off.data_ptr(), d_cnt.data_ptr(), 1,
                                               d_out.data_ptr(), cap, d_len.data_ptr(), d_st.data_ptr(),
                                               _native.stream_ptr()), "lpic_rc_encode_streams")
        if int(d_st.item()):
            raise RuntimeError(f"range encoder status {int(d_st.item())}")
        return d_out[:int(d_len.item())].cpu().numpy().tobytes()


class RangeDecoder:
    def __init__(self, data: bytes):
        L = _native.load()
        self._L = L
        buf = np.frombuffer(bytes(data), np.uint8)
        h = C.c_void_p()
        rc = L.lpic_rc_dec_create(buf.ctypes.data if buf.size else None, buf.size, C.byref(h))
        self._h = h.value
        if rc == _native.LPIC_S_CORRUPT:
            raise CorruptStreamError("compressed stream exhausted prematurely")
        _native.check(rc, "lpic_rc_dec_create")

    def decode(self, cdf) -> int:
        """Return the next symbol coded with this CDF table."""
        table = np.ascontiguousarray(cdf, dtype=np.int64)
        if table.shape != (257,):
            raise ValueError("expected a 257-entry cumulative table")
        sym = C.c_int32(0)
        rc = self._L.lpic_rc_dec_decode(self._h, table.ctypes.data, C.byref(sym))
        if rc == _native.LPIC_S_CORRUPT:
            raise CorruptStreamError("compressed stream exhausted prematurely")
        _native.check(rc, "lpic_rc_dec_decode")
        return int(sym.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._L.lpic_rc_dec_destroy(h)
            except Exception:
                pass


def rate_of(probabilities, symbol: int) -> float:
    """Ideal code length -log2(p[symbol]) in bits."""
    return float(-np.log2(probabilities[symbol]))
