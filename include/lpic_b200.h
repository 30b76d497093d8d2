/*
 * lpic_b200.h -- C-ABI of the B200-native LPIC hot path (liblpic_b200.so).
 *
 * This is the drop-in boundary for the reference package's hot path
 * (/root/reference/pkg/src/lpic).  The reference has no FFI of its own: its
 * "operator API" is the numba kernel seam in kernels.py plus the codec
 * entry points in codec.py.  Each entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - return value: 0 = ok, < 0 = LPIC_E_* error code (bad argument, CUDA
 *     failure, unsupported configuration).  Per-stream data errors are
 *     reported in a status word per image: LPIC_S_* bit flags.
 *   - "d_" pointers are device pointers on the model's device; "h_" pointers
 *     are host pointers (pageable or pinned).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     *_device entry points are asynchronous; host (h_) entry points
 *     synchronise the stream before returning.
 *   - modes: 0 = sequential, 1 = wavefront, 2 = diagonal
 *     (schedules.ScheduleMode, /root/reference/pkg/src/lpic/schedules.py:19-22).
 *   - precision: LPIC_PREC_COMPAT evaluates the network in the reference's
 *     canonical float32 order (bit-identical raw parameters, CPU-decodable
 *     streams); LPIC_PREC_FAST uses tcgen05 split-fp16 GEMMs (raw within
 *     1e-5 relative; streams decodable by this library in FAST mode only).
 */
#ifndef LPIC_B200_H
#define LPIC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lpic_model lpic_model_t;

/* return codes */
#define LPIC_OK 0
#define LPIC_E_ARG (-1)
#define LPIC_E_CUDA (-2)
#define LPIC_E_UNSUPPORTED (-3)
#define LPIC_E_NOMEM (-4)

/* per-image status flags */
#define LPIC_S_OK 0
#define LPIC_S_NONFINITE 1  /* codec.py:165-166  LpicError("network produced non-finite parameters") */
#define LPIC_S_CORRUPT 2    /* coder.py:94-95    CorruptStreamError */
#define LPIC_S_CAPACITY 4   /* output buffer too small */
#define LPIC_S_INTERNAL 8   /* a device-side pipeline stage never received its input (bounded wait expired) */

#define LPIC_PREC_COMPAT 0
#define LPIC_PREC_FAST 1

int lpic_version(void);
const char* lpic_last_error(void);

/* ---- model / weights ----------------------------------------------------
 * Replaces network.Weights + check_weights (network.py:85-164): uploads the
 * six float32 tensors (canonical storage order, HOST pointers) to the
 * current CUDA device and precomputes padded/split operand layouts.
 * dist: 0 Gaussian, 1 Logistic (network.Distribution, network.py:28-30). */
int lpic_model_create(const float* masked_w, const float* masked_b, const float* hidden_w,
                      const float* hidden_b, const float* out_w, const float* out_b,
                      int K, int C, int L, int h, int dist, lpic_model_t** out);
int lpic_model_destroy(lpic_model_t* m);
int lpic_model_set_precision(lpic_model_t* m, int precision);
/* network.weight_fingerprint (network.py:264-281): FNV-1a-64 of the LPWT
 * serialisation, computed natively at create time. */
uint64_t lpic_model_fingerprint(const lpic_model_t* m);
/* network.fnv1a64 (network.py:264-269) on an arbitrary host buffer */
uint64_t lpic_fnv1a64(const uint8_t* h_data, int64_t n);

/* ---- seam-level kernels (parity entry points) ---------------------------
 * kernels.forward_taps_f32 (kernels.py:117-136): d_taps (N,T,3) f32 -> d_raw (N,M) f32 */
int lpic_forward_taps(lpic_model_t* m, const float* d_taps, int64_t N, float* d_raw, void* stream);
/* kernels.forward_full_f32 (kernels.py:88-114): d_plane (H,W,3) f32 -> d_raw (H,W,M) f32 */
int lpic_forward_full(lpic_model_t* m, const float* d_plane, int H, int W, float* d_raw, void* stream);
/* kernels.channel_cdfs (kernels.py:296-313): d_raw (N,M) f32, d_rn/d_gn (N) f32
 * -> d_cdf (N,257) int32 (cdf[0]=0, cdf[256]=65536) */
int lpic_channel_cdfs(const float* d_raw, int64_t N, int M, int K, int dist, int channel,
                      const float* d_rn, const float* d_gn, int32_t* d_cdf, void* stream);
/* RangeEncoder over explicit streams (coder.py:30-73): stream s codes
 * d_sw[d_off[s] .. d_off[s]+d_cnt[s]) where each entry is start<<16 | (width-1);
 * bytes -> d_out + s*cap_each, length -> d_len[s]. */
int lpic_rc_encode_streams(const uint32_t* d_sw, const int64_t* d_off, const int64_t* d_cnt, int n_streams,
                           uint8_t* d_out, int64_t cap_each, int64_t* d_len, int32_t* d_status, void* stream);
/* RangeDecoder (coder.py:76-112): decode N symbols of one stream with
 * explicit tables d_cdf (N,257) int32 -> d_syms (N) int32 */
int lpic_rc_decode_tables(const uint8_t* d_data, int64_t len, const int32_t* d_cdf, int64_t N,
                          int32_t* d_syms, int32_t* d_status, void* stream);

/* kernels._quantized_cdf (kernels.py:250-293) from explicit mixture
 * parameters: d_pi, d_mu, d_s (N,K) f64 -> d_cdf (N,257) int32.  K <= 32.
 * Optional (NULL to skip): the kernel's scratch outputs as the reference
 * leaves them, d_pmf (N,256) f64 and d_neg_rem (N,256) f64 = floor - value. */
int lpic_quantized_cdf(const double* d_pi, const double* d_mu, const double* d_s, int64_t N, int K, int dist,
                       int32_t* d_cdf, double* d_pmf, double* d_neg_rem, void* stream);

/* coder.RangeDecoder (coder.py:76-112), the interactive one-symbol-per-call
 * API, as host code (a device round trip per symbol would cost ~500x the
 * work; the codec's own decoding runs on the GPU).  h_data is copied.
 * create/decode return 0, LPIC_S_CORRUPT (> 0) once the stream needed more
 * than 3 virtual zero bytes (CorruptStreamError), or an LPIC_E_* code. */
typedef struct lpic_rc_dec lpic_rc_dec_t;
int lpic_rc_dec_create(const uint8_t* h_data, int64_t len, lpic_rc_dec_t** out);
int lpic_rc_dec_decode(lpic_rc_dec_t* d, const int64_t* h_cdf /* 257 */, int32_t* h_sym);
int lpic_rc_dec_destroy(lpic_rc_dec_t* d);

/* kernels.true_symbol_probs (kernels.py:316-346): unquantised probability
 * of each coded symbol.  d_raw (N,M) f32, d_syms (N,3) int64, d_rn/d_gn (N)
 * f32 -> d_out (N,3) f64 */
int lpic_true_symbol_probs(const float* d_raw, int64_t N, int M, int K, int dist, const int64_t* d_syms,
                           const float* d_rn, const float* d_gn, double* d_out, void* stream);

/* ---- codec (batch) -------------------------------------------------------
 * codec.encode (codec.py:156-190) over n same-size images.
 * d_images (n,H,W,3) u8; payload of image b -> d_payload + b*cap_each,
 * length d_lens[b], status d_status[b].  Optional traces (CodecTrace,
 * codec.py:65-73) in coding order: d_trace_raw (n,H*W,M) f32,
 * d_trace_cdf (n,H*W,3,257) int32; pass NULL to skip. */
int lpic_encode_batch_device(lpic_model_t* m, const uint8_t* d_images, int n, int H, int W, int mode,
                             uint8_t* d_payload, int64_t cap_each, int64_t* d_lens, int32_t* d_status,
                             float* d_trace_raw, int32_t* d_trace_cdf, void* stream);
/* codec.decode (codec.py:193-247), the wavefront decoder, over n same-size
 * streams: payload b at d_payload + d_offs[b], length d_lens[b]. */
int lpic_decode_batch_device(lpic_model_t* m, const uint8_t* d_payload, const int64_t* d_offs,
                             const int64_t* d_lens, int n, int H, int W, int mode, uint8_t* d_images,
                             int32_t* d_status, float* d_trace_raw, int32_t* d_trace_cdf, void* stream);
/* Host-buffer variants (end-to-end: H2D, kernels, D2H inside the call).
 * encode: h_images (n,H,W,3) -> packed payloads in h_payload (capacity
 * payload_cap bytes), image b at h_offs[b], length h_lens[b]. */
int lpic_encode_batch(lpic_model_t* m, const uint8_t* h_images, int n, int H, int W, int mode,
                      uint8_t* h_payload, int64_t payload_cap, int64_t* h_offs, int64_t* h_lens,
                      int32_t* h_status, void* stream);
int lpic_decode_batch(lpic_model_t* m, const uint8_t* h_payload, const int64_t* h_offs,
                      const int64_t* h_lens, int n, int H, int W, int mode, uint8_t* h_images,
                      int32_t* h_status, void* stream);
/* The encoder's network stage alone (codec._raw_in_coding_order,
 * codec.py:116-145, in the model's precision): d_images (n,H,W,3) u8 ->
 * d_raw (n, H*W, 12K) f32 in coding order.  Used to time the network
 * kernel (compat: CUDA cores; FAST: tcgen05) on its own. */
int lpic_network_coding_order(lpic_model_t* m, const uint8_t* d_images, int n, int H, int W, int mode, float* d_raw,
                              void* stream);
/* codec.theoretical_bpsp (codec.py:255-274): -log2 of the unquantised
 * probability of every sub-pixel, in coding order: d_bits (n, H*W, 3) f64
 * (theoretical_bpsp = sum / (3HW)). */
int lpic_theoretical_bits(lpic_model_t* m, const uint8_t* d_images, int n, int H, int W, int mode, double* d_bits,
                          void* stream);
/* number of kernel launches issued by the last codec call (for bench accounting) */
int lpic_last_launch_count(const lpic_model_t* m);
/* training._mixture_loss (training.py:138-213), teacher forced, float64:
 * d_raw (N, 12K) f32 network outputs, d_images (N, 3) u8 -> d_logp (N) f64
 * = sum over r, g, b of log P(sub-pixel) (loss = -sum(d_logp) / (N ln 2)),
 * and, if d_draw is not null, d loss / d raw (N, 12K) f32. */
int lpic_mixture_loss_grad(const float* d_raw, const uint8_t* d_images, int64_t N, int K, int dist, double* d_logp,
                           float* d_draw, void* stream);
/* The same on float64 network outputs (the reference's float64 training
 * path, training.py:219-240, used by finite_difference_check). */
int lpic_mixture_loss_grad_f64(const double* d_raw, const uint8_t* d_images, int64_t N, int K, int dist,
                               double* d_logp, double* d_draw, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LPIC_B200_H */
