// lpic_train.cu -- the training loss of the desk-scale trainer on the GPU:
// teacher-forced discretised-mixture likelihood and its gradient with
// respect to the raw network outputs, fused per pixel.
//
// Restates training._mixture_loss (/root/reference/pkg/src/lpic/training.py:138-213)
// in float64, one thread per pixel:
//   log pi   = max-shifted log-softmax of the 3K logits
//   s        = exp(clip(rho, -7, 7))           (gradient gated to the open interval)
//   mu       = mu0 + tanh(c) * {rn, rn gn}      (rn, gn = (2 sym - 255) / 255 in float64)
//   P        = F((hi - mu)/s) - F((lo - mu)/s) on EDGES (+-inf at 0 / 255),
//              clamped at 1e-12 before the log
//   log p    = logsumexp_k(log pi_k + log P_k)  per channel, summed over r, g, b
// and the reference's hand-derived gradient (dlogits = (pi - q) / (N ln 2),
// dmu, drho, dcoef through tanh).  The network's own forward/backward are plain
// GEMMs (training.py:93-129) and run as library GEMMs from the host layer.
#include "../../include/lpic_b200.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

namespace {

constexpr int TR_KMAX = 16;
constexpr double TR_FLOOR = 1e-12;          // _BIN_PROB_FLOOR (training.py:31)
constexpr double TR_INV_SQRT_2PI = 0.3989422804014327;
constexpr double TR_LN2 = 0.6931471805599453;

__device__ __forceinline__ double edge(int k) { return (2.0 * (double)k - 256.0) / 255.0; }   // kernels.py:34

// F and f at z (training._cdf_pdf, training.py:128-135); z may be +-inf
__device__ __forceinline__ void cdf_pdf(double z, int dist, double& F, double& f) {
    if (dist == 0) {
        F = 0.5 * erfc(-z * 0.7071067811865476);          // ndtr
        f = isinf(z) ? 0.0 : exp(-0.5 * z * z) * TR_INV_SQRT_2PI;
    } else {
        F = 1.0 / (1.0 + exp(-z));                          // expit
        f = F * (1.0 - F);
    }
}

// R: float32 network outputs (the trainer) or float64 (the reference's
// float64 path: finite-difference checks)
template <typename R>
__global__ void __launch_bounds__(128)
k_mixture_loss(const R* __restrict__ raw, const uint8_t* __restrict__ images, int64_t N, int K, int dist,
               double* __restrict__ logp_out, R* __restrict__ draw) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int M = 12 * K;
    const R* r = raw + n * M;
    const int sym[3] = {images[3 * n], images[3 * n + 1], images[3 * n + 2]};
    const double rn = (2.0 * sym[0] - 255.0) / 255.0, gn = (2.0 * sym[1] - 255.0) / 255.0;
    const double scale = 1.0 / ((double)N * TR_LN2);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double tanhv[3][TR_KMAX];
    for (int c = 0; c < 3; c++)
        for (int k = 0; k < K; k++) tanhv[c][k] = tanh((double)r[9 * K + c * K + k]);
    double total = 0.0;
    double dmu_eff[3][TR_KMAX];
    for (int ch = 0; ch < 3; ch++) {
        // log-softmax of the logits (max-shifted)
        double lmax = -inf;
        for (int k = 0; k < K; k++) lmax = fmax(lmax, (double)r[ch * K + k]);
        double lsum = 0.0;
        for (int k = 0; k < K; k++) lsum += exp((double)r[ch * K + k] - lmax);
        const double llog = log(lsum);
        const int s = sym[ch];
        const double lo = s == 0 ? -inf : edge(s), hi = s == 255 ? inf : edge(s + 1);
        double joint[TR_KMAX], P[TR_KMAX], fl_[TR_KMAX], fu_[TR_KMAX], zl_[TR_KMAX], zu_[TR_KMAX], sd[TR_KMAX];
        bool open_s[TR_KMAX];
        double jmax = -inf;
        for (int k = 0; k < K; k++) {
            const double logpi = (double)r[ch * K + k] - lmax - llog;
            const double rho = (double)r[6 * K + ch * K + k];
            const double sv = exp(fmin(fmax(rho, -7.0), 7.0));
            double mu = (double)r[3 * K + ch * K + k];
            if (ch == 1) mu += tanhv[0][k] * rn;
            else if (ch == 2) mu += tanhv[1][k] * rn + tanhv[2][k] * gn;
            const double zl = (lo - mu) / sv, zu = (hi - mu) / sv;
            double Fl, fl, Fu, fu;
            cdf_pdf(zl, dist, Fl, fl);
            cdf_pdf(zu, dist, Fu, fu);
            P[k] = Fu - Fl;
            joint[k] = logpi + log(fmax(P[k], TR_FLOOR));
            jmax = fmax(jmax, joint[k]);
            fl_[k] = fl; fu_[k] = fu; zl_[k] = zl; zu_[k] = zu; sd[k] = sv;
            open_s[k] = rho > -7.0 && rho < 7.0;
        }
        double jsum = 0.0;
        for (int k = 0; k < K; k++) jsum += exp(joint[k] - jmax);
        const double logp = jmax + log(jsum);
        total += logp;
        if (draw) {
            R* d = draw + n * M;
            for (int k = 0; k < K; k++) {
                const double pi = exp((double)r[ch * K + k] - lmax - llog);
                const double q = exp(joint[k] - logp);
                d[ch * K + k] = (R)((pi - q) * scale);                                  // dlogits
                const double A = P[k] > TR_FLOOR ? q / fmax(P[k], TR_FLOOR) * scale : 0.0;
                const double dm = A * (fu_[k] - fl_[k]) / sd[k];
                dmu_eff[ch][k] = dm;
                d[3 * K + ch * K + k] = (R)dm;                                          // dmu
                const double zfl = isfinite(zl_[k]) ? zl_[k] * fl_[k] : 0.0;
                const double zfu = isfinite(zu_[k]) ? zu_[k] * fu_[k] : 0.0;
                d[6 * K + ch * K + k] = (R)(open_s[k] ? A * (zfu - zfl) : 0.0);         // drho
            }
        }
    }
    logp_out[n] = total;
    if (draw) {
        R* d = draw + n * M;
        for (int k = 0; k < K; k++) {                       // dcoef through tanh (training.py:199-203)
            d[9 * K + 0 * K + k] = (R)(dmu_eff[1][k] * rn * (1.0 - tanhv[0][k] * tanhv[0][k]));
            d[9 * K + 1 * K + k] = (R)(dmu_eff[2][k] * rn * (1.0 - tanhv[1][k] * tanhv[1][k]));
            d[9 * K + 2 * K + k] = (R)(dmu_eff[2][k] * gn * (1.0 - tanhv[2][k] * tanhv[2][k]));
        }
    }
}

}  // namespace

extern "C" int lpic_mixture_loss_grad(const float* d_raw, const uint8_t* d_images, int64_t N, int K, int dist,
                                      double* d_logp, float* d_draw, void* stream) {
    if (N < 0 || K < 1 || K > TR_KMAX || (dist != 0 && dist != 1) || !d_raw || !d_images || !d_logp)
        return LPIC_E_ARG;
    if (N == 0) return 0;
    k_mixture_loss<float><<<(unsigned)((N + 127) / 128), 128, 0, (cudaStream_t)stream>>>(d_raw, d_images, N, K, dist,
                                                                                         d_logp, d_draw);
    return cudaGetLastError() == cudaSuccess ? 0 : LPIC_E_CUDA;
}

extern "C" int lpic_mixture_loss_grad_f64(const double* d_raw, const uint8_t* d_images, int64_t N, int K, int dist,
                                          double* d_logp, double* d_draw, void* stream) {
    if (N < 0 || K < 1 || K > TR_KMAX || (dist != 0 && dist != 1) || !d_raw || !d_images || !d_logp)
        return LPIC_E_ARG;
    if (N == 0) return 0;
    k_mixture_loss<double><<<(unsigned)((N + 127) / 128), 128, 0, (cudaStream_t)stream>>>(d_raw, d_images, N, K,
                                                                                          dist, d_logp, d_draw);
    return cudaGetLastError() == cudaSuccess ? 0 : LPIC_E_CUDA;
}
