/*
 * lpic_oracle.c -- CPU restatement of the LPIC hot path.  TEST INFRASTRUCTURE
 * ONLY: the parity checker and the CPU baseline, never the product path.
 *
 * Build flags matter: -ffp-contract=off (the reference's numba kernels do
 * not contract a*b+c into FMA) and no -ffast-math.
 * Every function cites the reference unit it restates.
 */
#include "lpic_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CDF_TOTAL 65536
#define CDF_FLOOR_TOTAL (CDF_TOTAL - 256) /* kernels.py:37-38 */
static const double SQRT1_2 = 0.7071067811865476; /* kernels.py:40 */
static const float LEAKY = 0.01f;                  /* kernels.py:30 */

/* EDGES[k] = (2k - 256)/255 in float64 (kernels.py:34) */
static double EDGES[257];
static float NORM_LUT[256];
static int g_init = 0;
static void init_tables(void) {
    if (g_init) return;
    for (int k = 0; k < 257; k++) EDGES[k] = (2.0 * (double)k - 256.0) / 255.0;
    /* network.normalize: float32 x / 127.5f - 1.0f with true division (network.py:172-177) */
    for (int v = 0; v < 256; v++) {
        volatile float x = (float)v;
        volatile float q = x / 127.5f;
        NORM_LUT[v] = q - 1.0f;
    }
    g_init = 1;
}

float lpo_normalize_value(int v) { init_tables(); return NORM_LUT[v & 255]; }

/* kernels.causal_tap_offsets (kernels.py:42-55) */
int lpo_tap_count(int h) { return (2 * h + 1) * h + h; }
void lpo_tap_offsets(int h, int32_t *out) {
    int n = 0;
    for (int di = -h; di < 0; di++)
        for (int dj = -h; dj <= h; dj++) { out[2 * n] = di; out[2 * n + 1] = dj; n++; }
    for (int dj = -h; dj < 0; dj++) { out[2 * n] = 0; out[2 * n + 1] = dj; n++; }
}

/* ------------------------------------------------------------------------ */
/* network: masked layer + _dense_stack (kernels.py:63-136), canonical order */
/* ------------------------------------------------------------------------ */
static void forward_one(const lpo_weights *w, const float *tx, float *raw, float *a, float *z) {
    const int C = w->C, T = lpo_tap_count(w->h), M = 12 * w->K, NH = w->L - 2;
    for (int f = 0; f < C; f++) {
        float acc = 0.0f;
        for (int t = 0; t < T; t++)
            for (int c = 0; c < 3; c++) acc = acc + w->masked_w[(t * 3 + c) * C + f] * tx[t * 3 + c];
        acc = acc + w->masked_b[f];
        a[f] = (acc >= 0.0f) ? acc : LEAKY * acc;
    }
    for (int l = 0; l < NH; l++) {
        for (int o = 0; o < C; o++) {
            const float *wr = w->hidden_w + ((int64_t)l * C + o) * C;
            float acc = 0.0f;
            for (int i = 0; i < C; i++) acc = acc + wr[i] * a[i];
            acc = acc + w->hidden_b[l * C + o];
            z[o] = (acc >= 0.0f) ? acc : LEAKY * acc;
        }
        memcpy(a, z, sizeof(float) * C);
    }
    for (int m = 0; m < M; m++) {
        const float *wr = w->out_w + (int64_t)m * C;
        float acc = 0.0f;
        for (int i = 0; i < C; i++) acc = acc + wr[i] * a[i];
        raw[m] = acc + w->out_b[m];
    }
}

int lpo_forward_taps(const lpo_weights *w, const float *taps, int64_t N, float *out) {
    const int T = lpo_tap_count(w->h), M = 12 * w->K;
    float *a = (float *)malloc(sizeof(float) * w->C), *z = (float *)malloc(sizeof(float) * w->C);
    for (int64_t n = 0; n < N; n++) forward_one(w, taps + n * T * 3, out + n * M, a, z);
    free(a); free(z);
    return LPO_OK;
}

/* plain causal gather with zero padding (kernels.py:96-108) */
static void gather_plain(const float *plane, int H, int W, int h, int i, int j, float *tx) {
    int n = 0;
    for (int di = -h; di <= 0; di++) {
        int djmax = (di < 0) ? h : -1;
        for (int dj = -h; dj <= djmax; dj++, n++) {
            int ii = i + di, jj = j + dj;
            if (ii >= 0 && ii < H && jj >= 0 && jj < W) {
                const float *p = plane + ((int64_t)ii * W + jj) * 3;
                tx[n * 3 + 0] = p[0]; tx[n * 3 + 1] = p[1]; tx[n * 3 + 2] = p[2];
            } else {
                tx[n * 3 + 0] = 0.0f; tx[n * 3 + 1] = 0.0f; tx[n * 3 + 2] = 0.0f;
            }
        }
    }
}

int lpo_forward_full(const lpo_weights *w, const float *plane, int H, int W, float *out, int threads) {
    init_tables();
    const int T = lpo_tap_count(w->h), M = 12 * w->K;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        float *a = (float *)malloc(sizeof(float) * w->C), *z = (float *)malloc(sizeof(float) * w->C);
        float *tx = (float *)malloc(sizeof(float) * T * 3);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int i = 0; i < H; i++)
            for (int j = 0; j < W; j++) {
                gather_plain(plane, H, W, w->h, i, j, tx);
                forward_one(w, tx, out + ((int64_t)i * W + j) * M, a, z);
            }
        free(a); free(z); free(tx);
    }
    return LPO_OK;
}

/* ------------------------------------------------------------------------ */
/* mixture -> quantized CDF (kernels.py:202-313)                              */
/* ------------------------------------------------------------------------ */
static inline double cdf_value(double z, int dist) { /* kernels.py:202-209 */
    if (dist == 0) return 0.5 * erfc(-z * SQRT1_2);
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    double e = exp(z);
    return e / (1.0 + e);
}

/* kernels._channel_mixture (kernels.py:212-247).  Precision as numba types
 * it: softmax and scales in float64; the mean update in float32 with libm
 * tanhf, because raw/rn/gn are float32. */
static void channel_mixture(const float *raw, int K, int ch, float rn, float gn,
                            double *pi, double *mu, double *s) {
    const int base = ch * K;
    double m = -1.0e300;
    for (int i = 0; i < K; i++) { double v = (double)raw[base + i]; if (v > m) m = v; }
    double tot = 0.0;
    for (int i = 0; i < K; i++) { double e = exp((double)raw[base + i] - m); pi[i] = e; tot += e; }
    for (int i = 0; i < K; i++) pi[i] = pi[i] / tot;
    for (int i = 0; i < K; i++) {
        float v = raw[3 * K + base + i];
        if (ch == 1) {
            v = v + tanhf(raw[9 * K + i]) * rn;
        } else if (ch == 2) {
            v = v + tanhf(raw[10 * K + i]) * rn + tanhf(raw[11 * K + i]) * gn;
        }
        mu[i] = (double)v;
        double rho = (double)raw[6 * K + base + i];
        if (rho < -7.0) rho = -7.0;
        else if (rho > 7.0) rho = 7.0;
        s[i] = exp(rho);
    }
}

typedef struct { double key; int idx; } rem_t;
static int rem_cmp(const void *pa, const void *pb) {
    const rem_t *a = (const rem_t *)pa, *b = (const rem_t *)pb;
    int an = isnan(a->key), bn = isnan(b->key);
    if (an != bn) return an ? 1 : -1;               /* numpy sorts NaN last */
    if (!an) { if (a->key < b->key) return -1; if (a->key > b->key) return 1; }
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx); /* mergesort is stable */
}

/* quantization tail of kernels._quantized_cdf (kernels.py:272-293) */
static void quantize(const double *pmf, int64_t *cdf) {
    double total = 0.0;
    for (int k = 0; k < 256; k++) total += pmf[k];
    double scale = (double)CDF_FLOOR_TOTAL / total;
    int64_t acc = 0;
    rem_t rem[256];
    for (int k = 0; k < 256; k++) {
        double v = pmf[k] * scale;
        double f = floor(v);
        if (f > (double)CDF_FLOOR_TOTAL) f = (double)CDF_FLOOR_TOTAL;
        int64_t m = (int64_t)f + 1;
        cdf[k + 1] = m;
        rem[k].key = f - v;
        rem[k].idx = k;
        acc += m;
    }
    int64_t deficit = CDF_TOTAL - acc;
    if (deficit > 0) {
        qsort(rem, 256, sizeof(rem_t), rem_cmp);
        for (int64_t d = 0; d < deficit; d++) cdf[rem[d].idx + 1] += 1;
    }
    cdf[0] = 0;
    for (int k = 0; k < 256; k++) cdf[k + 1] += cdf[k];
}

void lpo_quantize_pmf(const double *pmf, int64_t *cdf) { quantize(pmf, cdf); }

/* kernels._quantized_cdf (kernels.py:250-293) */
static void quantized_cdf(const double *pi, const double *mu, const double *s, int K, int dist,
                          int64_t *cdf) {
    double pmf[256];
    for (int k = 0; k < 256; k++) pmf[k] = 0.0;
    for (int i = 0; i < K; i++) {
        double inv = 1.0 / s[i];
        double prev = 0.0;
        for (int k = 0; k < 256; k++) {
            double cur = (k == 255) ? 1.0 : cdf_value((EDGES[k + 1] - mu[i]) * inv, dist);
            double d = cur - prev;
            if (d > 0.0) pmf[k] += pi[i] * d;
            prev = cur;
        }
    }
    quantize(pmf, cdf);
}

static void table_for(const float *raw, int K, int dist, int ch, float rn, float gn, int64_t *cdf) {
    double pi[64], mu[64], s[64];
    channel_mixture(raw, K, ch, rn, gn, pi, mu, s);
    quantized_cdf(pi, mu, s, K, dist, cdf);
}

/* kernels.channel_cdfs (kernels.py:296-313) */
void lpo_channel_cdfs(const float *raw, int64_t N, int M, int K, int dist, int channel,
                      const float *rn, const float *gn, int64_t *out, int threads) {
    init_tables();
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (int64_t n = 0; n < N; n++)
        table_for(raw + n * M, K, dist, channel, rn[n], gn[n], out + n * 257);
}

/* kernels.true_symbol_probs (kernels.py:316-346) */
void lpo_true_symbol_probs(const float *raw, int64_t N, int M, const int64_t *syms,
                           const float *rn, const float *gn, int K, int dist, double *out) {
    init_tables();
    double pi[64], mu[64], s[64];
    for (int64_t n = 0; n < N; n++) {
        for (int ch = 0; ch < 3; ch++) {
            channel_mixture(raw + n * M, K, ch, rn[n], gn[n], pi, mu, s);
            int64_t x = syms[n * 3 + ch];
            double p = 0.0;
            for (int i = 0; i < K; i++) {
                double inv = 1.0 / s[i];
                double lo = (x == 0) ? 0.0 : cdf_value((EDGES[x] - mu[i]) * inv, dist);
                double hi = (x == 255) ? 1.0 : cdf_value((EDGES[x + 1] - mu[i]) * inv, dist);
                double d = hi - lo;
                if (d > 0.0) p += pi[i] * d;
            }
            out[n * 3 + ch] = p;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* range coder (coder.py:22-112)                                              */
/* ------------------------------------------------------------------------ */
#define RC_TOP (1ULL << 48)
#define RC_BOTTOM (1ULL << 40)
#define RC_MASK (RC_TOP - 1)

typedef struct { uint64_t low, range; uint8_t *out; int64_t n, cap; int err; } rc_enc;

static void rc_enc_init(rc_enc *e, uint8_t *out, int64_t cap) {
    e->low = 0; e->range = RC_TOP - 1; e->out = out; e->n = 0; e->cap = cap; e->err = 0;
}
static void rc_carry(rc_enc *e) { /* coder.py:52-57 */
    int64_t i = e->n - 1;
    while (i >= 0 && e->out[i] == 0xFF) { e->out[i] = 0; i--; }
    if (i >= 0) e->out[i] += 1; else e->err = LPO_ERR_ARG;
}
static void rc_put(rc_enc *e, uint8_t b) {
    if (e->n >= e->cap) { e->err = LPO_ERR_CAPACITY; return; }
    e->out[e->n++] = b;
}
static void rc_encode(rc_enc *e, uint32_t start, uint32_t width) { /* coder.py:37-50 */
    uint64_t r = e->range >> 16;
    e->low += r * start;
    e->range = r * width;
    if (e->low >= RC_TOP) { e->low -= RC_TOP; rc_carry(e); }
    while (e->range < RC_BOTTOM) {
        rc_put(e, (uint8_t)((e->low >> 40) & 0xFF));
        e->low = (e->low << 8) & RC_MASK;
        e->range <<= 8;
    }
}
static void rc_finish(rc_enc *e) { /* coder.py:59-73 */
    const int tail_bits = 48 - 24;
    uint64_t value = ((e->low + (1ULL << tail_bits) - 1) >> tail_bits) << tail_bits;
    if (value >= RC_TOP) { value -= RC_TOP; rc_carry(e); }
    for (int k = 0; k < 3; k++) rc_put(e, (uint8_t)((value >> (48 - 8 * (k + 1))) & 0xFF));
}

typedef struct { const uint8_t *data; int64_t len, pos; int virt; uint64_t range, code; int err; } rc_dec;

static int rc_next(rc_dec *d) { /* coder.py:86-96 */
    if (d->pos < d->len) return d->data[d->pos++];
    d->virt++;
    if (d->virt > 3) d->err = LPO_ERR_CORRUPT;
    return 0;
}
static void rc_dec_init(rc_dec *d, const uint8_t *data, int64_t len) {
    d->data = data; d->len = len; d->pos = 0; d->virt = 0; d->range = RC_TOP - 1; d->code = 0; d->err = 0;
    for (int k = 0; k < 6; k++) d->code = (d->code << 8) | (uint64_t)rc_next(d);
}
static int rc_decode(rc_dec *d, const int64_t *cdf) { /* coder.py:98-112 */
    uint64_t r = d->range >> 16;
    uint64_t target = d->code / r;
    if (target > 65535) target = 65535;
    int lo = 0, hi = 256; /* largest s with cdf[s] <= target */
    while (hi - lo > 1) { int mid = (lo + hi) >> 1; if ((uint64_t)cdf[mid] <= target) lo = mid; else hi = mid; }
    uint64_t start = (uint64_t)cdf[lo], width = (uint64_t)(cdf[lo + 1] - cdf[lo]);
    d->code -= r * start;
    d->range = r * width;
    while (d->range < RC_BOTTOM) {
        d->code = ((d->code << 8) & RC_MASK) | (uint64_t)rc_next(d);
        d->range <<= 8;
    }
    return lo;
}

int lpo_rc_encode(const int32_t *syms, const int64_t *tables, int64_t N, uint8_t *out, int64_t cap,
                  int64_t *out_len) {
    rc_enc e;
    rc_enc_init(&e, out, cap);
    for (int64_t n = 0; n < N; n++) {
        const int64_t *cdf = tables + n * 257;
        int s = syms[n];
        rc_encode(&e, (uint32_t)cdf[s], (uint32_t)(cdf[s + 1] - cdf[s]));
    }
    rc_finish(&e);
    *out_len = e.n;
    return e.err;
}

int lpo_rc_decode(const uint8_t *data, int64_t len, const int64_t *tables, int64_t N, int32_t *syms_out) {
    rc_dec d;
    rc_dec_init(&d, data, len);
    for (int64_t n = 0; n < N && !d.err; n++) syms_out[n] = rc_decode(&d, tables + n * 257);
    return d.err;
}

/* ------------------------------------------------------------------------ */
/* schedules (schedules.py:72-133)                                            */
/* ------------------------------------------------------------------------ */
int64_t lpo_step_count(int mode, int H, int W, int h) {
    if (mode == 0) return (int64_t)H * W;
    if (mode == 1) return (int64_t)(h + 1) * (H - 1) + W;
    return (int64_t)H + W - 1;
}

int64_t lpo_coding_order(int mode, int H, int W, int h, int32_t *order) {
    int64_t n = 0, passes = 0;
    if (mode == 0) {
        for (int i = 0; i < H; i++)
            for (int j = 0; j < W; j++) { order[2 * n] = i; order[2 * n + 1] = j; n++; }
        return (int64_t)H * W;
    }
    int64_t steps = lpo_step_count(mode, H, W, h);
    int a = (mode == 1) ? (h + 1) : 1; /* pixel (i,j) sits in step a*i + j */
    for (int64_t t = 0; t < steps; t++) {
        int any = 0;
        for (int i = 0; i < H; i++) {
            int64_t j = t - (int64_t)a * i;
            if (j < 0) break;
            if (j >= W) continue;
            order[2 * n] = i; order[2 * n + 1] = (int32_t)j; n++; any = 1;
        }
        passes += any;
    }
    return passes;
}

/* codec.gather_tap_values with schedules.diagonal substitutions
 * (codec.py:83-108, schedules.py:99-133) */
void lpo_gather_taps(const float *plane, int H, int W, int h, int mode, int i, int j, float *tx) {
    gather_plain(plane, H, W, h, i, j, tx);
    if (mode != 2) return;
    /* DIAGONAL_UNAVAILABLE = (-1,1), (-1,2), (-2,2); source (i-2, j+1) (schedules.py:44-45) */
    static const int un[3][2] = {{-1, 1}, {-1, 2}, {-2, 2}};
    int32_t taps[64 * 2];
    int T = lpo_tap_count(h);
    lpo_tap_offsets(h, taps);
    for (int u = 0; u < 3; u++) {
        int ti = i + un[u][0], tj = j + un[u][1];
        if (!(ti >= 0 && ti < H && tj >= 0 && tj < W)) continue;
        int k = 0;
        while (!(taps[2 * k] == un[u][0] && taps[2 * k + 1] == un[u][1])) k++;
        int si = i - 2, sj = j + 1, found = 0;
        if (!(si >= 0 && si < H && sj >= 0 && sj < W)) {
            for (int q = 0; q < T; q++) {
                int ci = i + taps[2 * q], cj = j + taps[2 * q + 1];
                if (ci >= 0 && ci < H && cj >= 0 && cj < W && ci + cj < i + j) { si = ci; sj = cj; found = 1; break; }
            }
        } else found = 1;
        for (int c = 0; c < 3; c++)
            tx[k * 3 + c] = found ? plane[((int64_t)si * W + sj) * 3 + c] : 0.0f;
    }
}

/* ------------------------------------------------------------------------ */
/* codec (codec.py:156-247)                                                   */
/* ------------------------------------------------------------------------ */
static int encode_prefix(const lpo_weights *w, const uint8_t *image, int H, int W, int mode,
                         uint8_t *payload, int64_t cap, int64_t *payload_len,
                         float *trace_raw, int64_t *trace_cdfs, int threads, int64_t max_px) {
    init_tables();
    const int64_t NF = (int64_t)H * W;
    const int64_t N = (max_px >= 0 && max_px < NF) ? max_px : NF; /* pixels coded (coding order) */
    const int M = 12 * w->K, T = lpo_tap_count(w->h);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * 2 * NF);
    float *plane = (float *)malloc(sizeof(float) * 3 * NF);
    uint32_t *sw = (uint32_t *)malloc(sizeof(uint32_t) * 2 * 3 * N);
    int nonfinite = 0;
    lpo_coding_order(mode, H, W, w->h, order);
    for (int64_t p = 0; p < 3 * NF; p++) plane[p] = NORM_LUT[image[p]];
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads) reduction(| : nonfinite)
#endif
    {
        float *a = (float *)malloc(sizeof(float) * w->C), *z = (float *)malloc(sizeof(float) * w->C);
        float tx[64 * 3], raw[12 * 64];
        int64_t cdf[257];
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t n = 0; n < N; n++) {
            int i = order[2 * n], j = order[2 * n + 1];
            lpo_gather_taps(plane, H, W, w->h, mode, i, j, tx);
            forward_one(w, tx, raw, a, z);
            for (int m = 0; m < M; m++) if (!isfinite(raw[m])) nonfinite = 1;
            if (trace_raw) memcpy(trace_raw + n * M, raw, sizeof(float) * M);
            const uint8_t *px = image + ((int64_t)i * W + j) * 3;
            float rn = NORM_LUT[px[0]], gn = NORM_LUT[px[1]];
            for (int ch = 0; ch < 3; ch++) {
                table_for(raw, w->K, w->dist, ch, ch >= 1 ? rn : 0.0f, ch == 2 ? gn : 0.0f, cdf);
                int s = px[ch];
                sw[(n * 3 + ch) * 2 + 0] = (uint32_t)cdf[s];
                sw[(n * 3 + ch) * 2 + 1] = (uint32_t)(cdf[s + 1] - cdf[s]);
                if (trace_cdfs) memcpy(trace_cdfs + (n * 3 + ch) * 257, cdf, sizeof(cdf));
            }
        }
        free(a); free(z);
    }
    (void)T;
    int err = LPO_OK;
    if (nonfinite) err = LPO_ERR_NONFINITE;
    else {
        rc_enc e;
        rc_enc_init(&e, payload, cap);
        for (int64_t q = 0; q < 3 * N; q++) rc_encode(&e, sw[2 * q], sw[2 * q + 1]);
        rc_finish(&e);
        *payload_len = e.n;
        err = e.err;
    }
    free(order); free(plane); free(sw);
    return err;
}

static int decode_prefix(const lpo_weights *w, const uint8_t *payload, int64_t payload_len,
                         int H, int W, int mode, uint8_t *image, float *trace_raw, int64_t *trace_cdfs,
                         int64_t max_px) {
    init_tables();
    const int64_t N = (int64_t)H * W;
    const int64_t stop = (max_px >= 0 && max_px < N) ? max_px : N;
    const int M = 12 * w->K;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * 2 * N);
    float *plane = (float *)calloc(3 * N, sizeof(float));
    float *a = (float *)malloc(sizeof(float) * w->C), *z = (float *)malloc(sizeof(float) * w->C);
    float tx[64 * 3], raw[12 * 64];
    int64_t cdf[257];
    lpo_coding_order(mode, H, W, w->h, order);
    memset(image, 0, 3 * N);
    rc_dec d;
    rc_dec_init(&d, payload, payload_len);
    for (int64_t n = 0; n < stop && !d.err; n++) {
        int i = order[2 * n], j = order[2 * n + 1];
        lpo_gather_taps(plane, H, W, w->h, mode, i, j, tx);
        forward_one(w, tx, raw, a, z);
        if (trace_raw) memcpy(trace_raw + n * M, raw, sizeof(float) * M);
        float rn = 0.0f, gn = 0.0f;
        int sym[3];
        for (int ch = 0; ch < 3; ch++) {
            table_for(raw, w->K, w->dist, ch, rn, gn, cdf);
            sym[ch] = rc_decode(&d, cdf);
            if (trace_cdfs) memcpy(trace_cdfs + (n * 3 + ch) * 257, cdf, sizeof(cdf));
            if (ch == 0) rn = NORM_LUT[sym[0]];
            if (ch == 1) gn = NORM_LUT[sym[1]];
        }
        uint8_t *px = image + ((int64_t)i * W + j) * 3;
        float *pp = plane + ((int64_t)i * W + j) * 3;
        for (int c = 0; c < 3; c++) { px[c] = (uint8_t)sym[c]; pp[c] = NORM_LUT[sym[c]]; }
    }
    int err = d.err;
    free(order); free(plane); free(a); free(z);
    return err;
}

int lpo_encode(const lpo_weights *w, const uint8_t *image, int H, int W, int mode,
               uint8_t *payload, int64_t cap, int64_t *payload_len,
               float *trace_raw, int64_t *trace_cdfs, int threads) {
    return encode_prefix(w, image, H, W, mode, payload, cap, payload_len, trace_raw, trace_cdfs, threads, -1);
}

/* CPU-baseline helper: a valid stream of the first max_px pixels (coding
 * order) of each image; its prefix decodes exactly like the full stream's. */
int lpo_encode_batch_prefix(const lpo_weights *w, const uint8_t *images, int n, int H, int W, int mode,
                            int64_t max_px, uint8_t *payloads, int64_t cap_each, int64_t *lens, int threads) {
    int err = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1) reduction(| : err)
#endif
    for (int b = 0; b < n; b++)
        err |= encode_prefix(w, images + (int64_t)b * H * W * 3, H, W, mode, payloads + (int64_t)b * cap_each,
                             cap_each, lens + b, NULL, NULL, 1, max_px);
    return err ? LPO_ERR_ARG : LPO_OK;
}

int lpo_decode(const lpo_weights *w, const uint8_t *payload, int64_t payload_len,
               int H, int W, int mode, uint8_t *image, float *trace_raw, int64_t *trace_cdfs) {
    return decode_prefix(w, payload, payload_len, H, W, mode, image, trace_raw, trace_cdfs, -1);
}

/* CPU-baseline sample: decode only the first max_px pixels (coding order) of
 * each stream, one stream per thread. */
int lpo_decode_batch_prefix(const lpo_weights *w, const uint8_t *payloads, int64_t cap_each, const int64_t *lens,
                            int n, int H, int W, int mode, int64_t max_px, uint8_t *images, int threads) {
    int err = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1) reduction(| : err)
#endif
    for (int b = 0; b < n; b++)
        err |= decode_prefix(w, payloads + (int64_t)b * cap_each, lens[b], H, W, mode,
                             images + (int64_t)b * H * W * 3, NULL, NULL, max_px);
    return err ? LPO_ERR_CORRUPT : LPO_OK;
}

int lpo_encode_batch(const lpo_weights *w, const uint8_t *images, int n, int H, int W, int mode,
                     uint8_t *payloads, int64_t cap_each, int64_t *lens, int threads) {
    int err = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1) reduction(| : err)
#endif
    for (int b = 0; b < n; b++)
        err |= lpo_encode(w, images + (int64_t)b * H * W * 3, H, W, mode, payloads + (int64_t)b * cap_each,
                          cap_each, lens + b, NULL, NULL, 1);
    return err ? LPO_ERR_ARG : LPO_OK;
}

int lpo_decode_batch(const lpo_weights *w, const uint8_t *payloads, int64_t cap_each, const int64_t *lens,
                     int n, int H, int W, int mode, uint8_t *images, int threads) {
    int err = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1) reduction(| : err)
#endif
    for (int b = 0; b < n; b++)
        err |= lpo_decode(w, payloads + (int64_t)b * cap_each, lens[b], H, W, mode,
                          images + (int64_t)b * H * W * 3, NULL, NULL);
    return err ? LPO_ERR_CORRUPT : LPO_OK;
}

/* network.fnv1a64 (network.py:264-269) */
uint64_t lpo_fnv1a64(const uint8_t *data, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < n; i++) { h ^= data[i]; h *= 0x100000001b3ULL; }
    return h;
}
