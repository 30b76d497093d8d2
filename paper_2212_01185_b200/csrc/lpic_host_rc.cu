// lpic_host_rc.cu -- the interactive range DECODER of the public coder API
// (coder.RangeDecoder, /root/reference/pkg/src/lpic/coder.py:76-112).
//
// RangeDecoder.decode(cdf) returns one symbol per call and the caller picks
// the next table from it (update_means, tests/test_coder.py), so the API is
// inherently one symbol at a time on the caller's thread: a device round
// trip per symbol would cost ~10 us of launch + sync for ~20 ns of work.
// This object is therefore host code, compiled into liblpic_b200.so next to
// the device decoder whose arithmetic it repeats (RcDecoder, lpic_rc.cuh);
// the codec's decode path never uses it -- streams are decoded on the GPU
// (k_decode2).  The matching encoder side (coder.RangeEncoder) collects the
// symbols and codes them on the GPU at finish() (lpic_rc_encode_streams).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/lpic_b200.h"

namespace {
constexpr uint64_t TOP = 1ull << 48;
constexpr uint64_t BOTTOM = 1ull << 40;
constexpr uint64_t MASK = TOP - 1;
}  // namespace

struct lpic_rc_dec {
    uint8_t* data;
    int64_t len, pos;
    int virt;
    uint64_t code, range;
    int status;
    int next_byte() {                         // coder.py:86-96: <= 3 virtual zero bytes
        if (pos < len) return data[pos++];
        virt++;
        if (virt > 3) status |= LPIC_S_CORRUPT;
        return 0;
    }
};

extern "C" {

int lpic_rc_dec_create(const uint8_t* h_data, int64_t len, lpic_rc_dec_t** out) {
    if (!out || len < 0 || (len > 0 && !h_data)) return LPIC_E_ARG;
    lpic_rc_dec* d = new (std::nothrow) lpic_rc_dec();
    if (!d) return LPIC_E_NOMEM;
    d->data = static_cast<uint8_t*>(std::malloc(len > 0 ? (size_t)len : 1));
    if (!d->data) { delete d; return LPIC_E_NOMEM; }
    if (len > 0) std::memcpy(d->data, h_data, (size_t)len);
    d->len = len; d->pos = 0; d->virt = 0; d->status = 0;
    d->range = TOP - 1; d->code = 0;
    for (int k = 0; k < 6; k++) d->code = (d->code << 8) | (uint64_t)d->next_byte();
    *out = d;
    return d->status ? LPIC_S_CORRUPT : LPIC_OK;
}

int lpic_rc_dec_decode(lpic_rc_dec_t* d, const int64_t* h_cdf, int32_t* h_sym) {
    if (!d || !h_cdf || !h_sym) return LPIC_E_ARG;
    const uint64_t r = d->range >> 16;
    uint64_t target = d->code / r;                        // coder.py:100-103
    if (target > 65535) target = 65535;
    // searchsorted(cdf, target, 'right') - 1 over the 257 entries (coder.py:104)
    int lo = 0, hi = 257;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint64_t)h_cdf[mid] <= target) lo = mid + 1; else hi = mid;
    }
    const int sym = lo - 1;
    if (sym < 0 || sym > 255) return LPIC_E_ARG;          // not a valid table for this target
    const uint64_t start = (uint64_t)h_cdf[sym], width = (uint64_t)(h_cdf[sym + 1] - h_cdf[sym]);
    d->code -= r * start;                                  // coder.py:107-111
    d->range = r * width;
    while (d->range < BOTTOM) {
        d->code = ((d->code << 8) & MASK) | (uint64_t)d->next_byte();
        d->range <<= 8;
    }
    *h_sym = sym;
    return d->status ? LPIC_S_CORRUPT : LPIC_OK;
}

int lpic_rc_dec_destroy(lpic_rc_dec_t* d) {
    if (d) {
        std::free(d->data);
        delete d;
    }
    return 0;
}

}  // extern "C"
