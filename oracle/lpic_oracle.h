/*
 * lpic_oracle.h -- CPU restatement of the LPIC hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle, not the product.  Only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load it.
 * It restates, in plain C with IEEE float32/float64 arithmetic and no FMA
 * contraction, the reference package's algorithm:
 *
 *   network      /root/reference/pkg/src/lpic/kernels.py:63-136
 *   mixture/CDF  /root/reference/pkg/src/lpic/kernels.py:202-313
 *   rate         /root/reference/pkg/src/lpic/kernels.py:316-346
 *   range coder  /root/reference/pkg/src/lpic/coder.py:30-112
 *   schedules    /root/reference/pkg/src/lpic/schedules.py:72-133
 *   codec        /root/reference/pkg/src/lpic/codec.py:83-247
 *   fingerprint  /root/reference/pkg/src/lpic/network.py:264-281
 *
 * Transcendentals come from the host libm (glibc erfc/exp/tanhf), which is
 * what the reference's numba kernels call.  Pinned against golden vectors
 * produced by running the reference itself (tests/golden/, made by
 * oracle/gen_golden.py).
 */
#ifndef LPIC_ORACLE_H
#define LPIC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int K, C, L, h, dist;       /* mixtures, filters, layers, kernel_half, distribution */
    const float *masked_w;      /* (T,3,C) */
    const float *masked_b;      /* (C)     */
    const float *hidden_w;      /* (L-2,C,C) out x in */
    const float *hidden_b;      /* (L-2,C) */
    const float *out_w;         /* (M,C)   */
    const float *out_b;         /* (M)     */
} lpo_weights;

/* error codes (mirrors include/lpic_b200.h) */
#define LPO_OK 0
#define LPO_ERR_ARG (-1)
#define LPO_ERR_NONFINITE (-2)
#define LPO_ERR_CORRUPT (-3)
#define LPO_ERR_CAPACITY (-4)

int lpo_tap_count(int h);
void lpo_tap_offsets(int h, int32_t *out /* (T,2) */);
float lpo_normalize_value(int v);

/* network: forward from gathered taps (N,T,3) -> (N,M) */
int lpo_forward_taps(const lpo_weights *w, const float *taps, int64_t N, float *out);
/* network: whole plane (H,W,3) normalized -> (H,W,M) */
int lpo_forward_full(const lpo_weights *w, const float *plane, int H, int W, float *out, int threads);

/* kernels.channel_cdfs: raw (N,M) f32, rn/gn (N) f32 -> out (N,257) int64 */
void lpo_channel_cdfs(const float *raw, int64_t N, int M, int K, int dist, int channel,
                      const float *rn, const float *gn, int64_t *out, int threads);
/* kernels.true_symbol_probs: syms (N,3) int64 -> out (N,3) f64 */
void lpo_true_symbol_probs(const float *raw, int64_t N, int M, const int64_t *syms,
                           const float *rn, const float *gn, int K, int dist, double *out);

/* mixture.quantize_cdf on an arbitrary pmf (256) -> cdf (257) */
void lpo_quantize_pmf(const double *pmf, int64_t *cdf);

/* range coder on explicit (symbol, table) streams */
int lpo_rc_encode(const int32_t *syms, const int64_t *tables /* (N,257) */, int64_t N,
                  uint8_t *out, int64_t cap, int64_t *out_len);
int lpo_rc_decode(const uint8_t *data, int64_t len, const int64_t *tables, int64_t N,
                  int32_t *syms_out);

/* schedules */
int64_t lpo_step_count(int mode, int H, int W, int h);
/* coding order (N,2) as (i,j) in bitstream order; returns number of non-empty steps */
int64_t lpo_coding_order(int mode, int H, int W, int h, int32_t *order_out);
/* gather taps for pixel (i,j) from a normalized plane with diag substitutions */
void lpo_gather_taps(const float *plane, int H, int W, int h, int mode, int i, int j, float *taps_out);

/* codec */
int lpo_encode(const lpo_weights *w, const uint8_t *image, int H, int W, int mode,
               uint8_t *payload, int64_t cap, int64_t *payload_len,
               float *trace_raw /* (N,M) or NULL */, int64_t *trace_cdfs /* (N,3,257) or NULL */,
               int threads);
int lpo_decode(const lpo_weights *w, const uint8_t *payload, int64_t payload_len,
               int H, int W, int mode, uint8_t *image_out,
               float *trace_raw, int64_t *trace_cdfs);
/* batch helpers for the CPU baseline: one image per thread */
int lpo_encode_batch(const lpo_weights *w, const uint8_t *images, int n, int H, int W, int mode,
                     uint8_t *payloads, int64_t cap_each, int64_t *lens, int threads);
int lpo_decode_batch(const lpo_weights *w, const uint8_t *payloads, int64_t cap_each,
                     const int64_t *lens, int n, int H, int W, int mode, uint8_t *images,
                     int threads);

int lpo_encode_batch_prefix(const lpo_weights *w, const uint8_t *images, int n, int H, int W, int mode,
                            int64_t max_px, uint8_t *payloads, int64_t cap_each, int64_t *lens, int threads);
int lpo_decode_batch_prefix(const lpo_weights *w, const uint8_t *payloads, int64_t cap_each,
                            const int64_t *lens, int n, int H, int W, int mode, int64_t max_px,
                            uint8_t *images, int threads);

uint64_t lpo_fnv1a64(const uint8_t *data, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
