// lpic_rc.cuh -- 48-bit range coder lanes, byte-compatible with the
// reference RangeEncoder / RangeDecoder (/root/reference/pkg/src/lpic/coder.py:22-112).
//
// The encoder keeps the reference's carry semantics without random access
// to already-written output: the emitted stream is F ++ [cache] ++ [0xFF]*nff
// where F is final, `cache` is the last byte a carry can still increment and
// the trailing 0xFF run is what coder.py:52-57 would zero on a carry.  This
// is exactly the reference's byte array, produced strictly sequentially.
#pragma once
#include <cstdint>

namespace lpic {

constexpr uint64_t RC_TOP = 1ull << 48;
constexpr uint64_t RC_BOTTOM = 1ull << 40;
constexpr uint64_t RC_MASK = RC_TOP - 1;

enum : int { ST_OK = 0, ST_NONFINITE = 1, ST_CORRUPT = 2, ST_CAPACITY = 4, ST_ARG = 8 };

struct RcEncoder {
    uint64_t low, range;
    uint8_t* out;
    int64_t pos, cap;
    uint32_t nff;
    int cache;        // -1: no byte emitted yet
    int status;

    __device__ __forceinline__ void init(uint8_t* o, int64_t c) {
        low = 0; range = RC_TOP - 1; out = o; pos = 0; cap = c; nff = 0; cache = -1; status = ST_OK;
    }
    __device__ __forceinline__ void put(int b, bool writer) {
        if (pos < cap) { if (writer) out[pos] = (uint8_t)b; }
        else status |= ST_CAPACITY;
        pos++;
    }
    __device__ __forceinline__ void emit(int b, bool writer) {
        if (cache < 0) { cache = b; return; }
        if (b == 0xFF) { nff++; return; }
        put(cache, writer);
        for (; nff; nff--) put(0xFF, writer);
        cache = b;
    }
    __device__ __forceinline__ void carry(bool writer) {   // coder.py:52-57
        if (nff) {
            put(cache + 1, writer);
            for (uint32_t q = 1; q < nff; q++) put(0x00, writer);
            cache = 0x00;
            nff = 0;
        } else {
            cache += 1;
        }
    }
    // coder.py:37-50
    __device__ __forceinline__ void encode(uint32_t start, uint32_t width, bool writer) {
        const uint64_t r = range >> 16;
        low += r * start;
        range = r * width;
        if (low >= RC_TOP) { low -= RC_TOP; carry(writer); }
        while (range < RC_BOTTOM) {
            emit((int)((low >> 40) & 0xFF), writer);
            low = (low << 8) & RC_MASK;
            range <<= 8;
        }
    }
    // coder.py:59-73
    __device__ __forceinline__ int64_t finish(bool writer) {
        uint64_t value = ((low + (1ull << 24) - 1) >> 24) << 24;
        if (value >= RC_TOP) { value -= RC_TOP; carry(writer); }
        for (int k = 0; k < 3; k++) emit((int)((value >> (40 - 8 * k)) & 0xFF), writer);
        if (cache >= 0) put(cache, writer);
        for (; nff; nff--) put(0xFF, writer);
        return pos;
    }
};

struct RcDecoder {
    uint64_t code, range;
    const uint8_t* data;
    int64_t len, pos;
    int virt;
    int status;
    uint32_t nb;      // advance_bf: bytes pos, pos+1 (0 past the end), loaded one advance ahead

    __device__ __forceinline__ int next_byte() {           // coder.py:86-96
        if (pos < len) return __ldg(data + pos++);
        virt++;
        if (virt > 3) status |= ST_CORRUPT;
        return 0;
    }
    __device__ __forceinline__ void init(const uint8_t* d, int64_t n) {
        data = d; len = n; pos = 0; virt = 0; status = ST_OK; range = RC_TOP - 1; code = 0;
        for (int k = 0; k < 6; k++) code = (code << 8) | (uint64_t)next_byte();
        prefetch2();
    }
    __device__ __forceinline__ void prefetch2() {
        nb = (pos < len ? (uint32_t)__ldg(data + pos) : 0u) | ((pos + 1 < len ? (uint32_t)__ldg(data + pos + 1) : 0u) << 8);
    }
    // target = min(code // r, 65535) (coder.py:100-103), exact: a float64
    // quotient estimate (code < 2^48, 2^24 <= r < 2^32, so q < 2^24 and the
    // refined reciprocal is off by far less than one unit) plus one integer
    // correction each way.
    __device__ __forceinline__ uint32_t target(uint64_t& r_out) const {
        const uint64_t r = range >> 16;
        const double rd = (double)r;
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rd));
        y = __fma_rn(y, __fma_rn(-rd, y, 1.0), y);
        uint64_t q = (uint64_t)__dmul_rz((double)code, y);
        if (q * r > code) q--;
        else if ((q + 1) * r <= code) q++;
        r_out = r;
        return q > 65535 ? 65535u : (uint32_t)q;
    }
    __device__ __forceinline__ void advance(uint64_t r, uint32_t start, uint32_t width) {   // coder.py:107-111
        code -= r * start;
        range = r * width;
        while (range < RC_BOTTOM) {
            code = ((code << 8) & RC_MASK) | (uint64_t)next_byte();
            range <<= 8;
        }
    }
    // The same, branch-free (so it can be scheduled into the shadow of other
    // work): r >= 2^24 and width >= 1 bound the renormalisation to two bytes.
    // The two bytes it may consume were loaded by the previous advance
    // (prefetch2), so no global load sits on the decoder chain's critical
    // path (in situ, r2q: the advance + target cost ~640 cycles per table
    // while the byte loads were issued inside it; ~50 with L1-resident data).
    __device__ __forceinline__ void advance_bf(uint64_t r, uint32_t start, uint32_t width) {
        code -= r * start;
        const uint64_t rg = r * width;
        const bool n1 = rg < RC_BOTTOM, n2 = rg < (RC_BOTTOM >> 8);
        const bool in0 = pos < len, in1 = pos + 1 < len;
        const uint64_t b0 = nb & 0xFFu, b1 = (nb >> 8) & 0xFFu;   // (0 past the end)
        virt += (int)(n1 && !in0) + (int)(n2 && !in1);        // bytes past the end read as 0
        status |= virt > 3 ? ST_CORRUPT : 0;                 // coder.py:94-95
        code = n2 ? (((code << 16) & RC_MASK) | (b0 << 8) | b1) : (n1 ? (((code << 8) & RC_MASK) | b0) : code);
        range = n2 ? rg << 16 : (n1 ? rg << 8 : rg);
        pos += (int64_t)n1 + (int64_t)n2;
        prefetch2();                                         // consumed by the next advance, a table later
    }
};

}  // namespace lpic
