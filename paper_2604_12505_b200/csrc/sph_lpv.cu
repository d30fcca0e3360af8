// LPV surrogate identification on the GPU (paper Sec. 4, and Sec. 5.3,
// P:423-446).  Self-scheduled LPV-SS model with affine scheduling (Eqs. surrogate_form,
// LPVparametrization), benchmark dimensions n_x = 4, n_u = 3, n_y = 3, n_p = 1, D = 0:
//   z_k = [x_k; u_k],  h1 = tanh(W1 z + b1),  h2 = tanh(W2 h1 + b2),  p_k = W3 h2 + b3
//   A = A0 + p A1,  B = B0 + p B1,  C = C0 + p C1
//   y^_k = C x_k,   x_{k+1} = A x_k + B u_k
// Objective (Eqs. pem, surrogate_optimization, regularization; reading LPV3 for S sequences):
//   F = 1/S sum_s 1/K sum_k ||y_sk - y^_sk||^2 + sigma2/2 ||theta||^2 + sigmax/2 sum_s ||x0_s||^2
// The gradient ("computed using automatic differentiation") is reverse mode written out:
// a forward sweep stores x_k, the backward sweep carries the adjoint lam_k = dF/dx_k
//   dy_k  = 2/(K S) (y^_k - y_k)
//   dA += lam_{k+1} x_k^T, dB += lam_{k+1} u_k^T, dC += dy_k x_k^T   (M0 gets d., M1 gets p d.)
//   dp    = <A1, dA> + <B1, dB> + <C1, dC>  -> back through the two tanh layers
//   lam_k = A^T lam_{k+1} + C^T dy_k + (W1^T da1)[0:4]
// The recurrence is sequential in k, so its latency sets the time: one quad of lanes per
// (restart r, sequence s) chain, all restarts and sequences of a training step in one launch (a
// CTA per restart, the per-sequence gradients summed in fixed order).  float64 throughout.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/sph.h"

namespace lpv {

constexpr int NX = 4, NU = 3, NY = 3, NH = 4, NZ = NX + NU;
constexpr int OA0 = 0, OB0 = 16, OC0 = 28, OA1 = 40, OB1 = 56, OC1 = 68;
constexpr int OW1 = 80, OB_1 = 108, OW2 = 112, OB_2 = 128, OW3 = 132, OB_3 = 136, NT = 137;
static_assert(NT == SPH_LPV_NTHETA, "parameter layout");
// Four lanes per (restart, sequence) chain: lane q owns row q of A, B, C (q < 3) and W1, neuron q
// of both tanh layers, and the gradients of exactly those parameters (registers, no spills).
// Vectors are exchanged inside the quad by shuffles; quad sums are butterflies, so every lane of
// a quad holds the same bits.  A CTA (one restart) runs 8 chains.
constexpr int LPV_T = 32;
constexpr int CH = LPV_T / 4;
constexpr unsigned FULL = 0xffffffffu;
constexpr int REC = 4 * NX + 1;   // per step and chain: x, h1, h2, y^ (one per lane), p

__device__ __forceinline__ double q4sum(double v) {
    v += __shfl_xor_sync(FULL, v, 1);
    return v + __shfl_xor_sync(FULL, v, 2);
}
__device__ __forceinline__ double q4get(double v, int j) { return __shfl_sync(FULL, v, j, 4); }
// tanh in float64 with a short dependency chain (the libm call branches and runs a long serial
// polynomial; here both halves run side by side and one is selected):
//   |a| < 1/8:  tanh x = x + x^3 P(x^2), Taylor to x^15 (truncation < 1e-17 relative)
//   else:       tanh x = (1 - t) / (1 + t), t = e^{-2x} = 2^n 2^f, 2^f by its Taylor series
//               to degree 13 on |f| <= 1/2 (Estrin), the quotient by a Newton-refined reciprocal
// Agreement with the libm tanh: a few ulp (tests compare the objective with the float64 oracle).
#ifndef SPH_LPV_FAST_TANH
#define SPH_LPV_FAST_TANH 1
#endif
__device__ __forceinline__ double tanh_d(double a) {
#if SPH_LPV_FAST_TANH
    const double x = fabs(a);
    const double x2 = x * x;
    double sm = fma(x2, -929569.0 / 638512875.0, 21844.0 / 6081075.0);
    sm = fma(x2, sm, -1382.0 / 155925.0);
    sm = fma(x2, sm, 62.0 / 2835.0);
    sm = fma(x2, sm, -17.0 / 315.0);
    sm = fma(x2, sm, 2.0 / 15.0);
    sm = fma(x2, sm, -1.0 / 3.0);
    sm = fma(x * x2, sm, x);
    const double z = fmax(-2.0 * 1.4426950408889634 * x, -1020.0);
    const double n = rint(z), f = z - n;
    const double f2 = f * f, f4 = f2 * f2, f8 = f4 * f4;
    // c_k = ln2^k / k!
    const double p01 = fma(f, 0.6931471805599453, 1.0);
    const double p23 = fma(f, 0.05550410866482158, 0.2402265069591007);
    const double p45 = fma(f, 0.0013333558146428443, 0.009618129107628477);
    const double p67 = fma(f, 1.525273380405984e-05, 0.00015403530393381606);
    const double p89 = fma(f, 1.0178086009239699e-07, 1.3215486790144307e-06);
    const double p1011 = fma(f, 4.4455382718708114e-10, 7.054911620801123e-09);
    const double p1213 = fma(f, 1.3691488853904124e-12, 2.5678435993488202e-11);
    const double q0 = fma(p23, f2, p01), q1 = fma(p67, f2, p45), q2 = fma(p1011, f2, p89);
    const double pw = fma(fma(p1213, f4, q2), f8, fma(q1, f4, q0));
    const double t = pw * __longlong_as_double((long long)((int)n + 1023) << 52);
    const double num = 1.0 - t, den = 1.0 + t;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    r = fma(r, fma(-den, r, 1.0), r);
    r = fma(r, fma(-den, r, 1.0), r);
    double qt = num * r;
    qt = fma(r, fma(-den, qt, num), qt);
    return copysign(x < 0.125 ? sm : qt, a);
#else
    return tanh(a);
#endif
}

__device__ __forceinline__ double pick4(const double* v, int q) {
    return q == 0 ? v[0] : q == 1 ? v[1] : q == 2 ? v[2] : v[3];
}

__global__ void __launch_bounds__(LPV_T) k_lpv(int R, int S, int K, const double* __restrict__ prm,
                                                const float* __restrict__ u,
                                                const float* __restrict__ y, double sigma2,
                                                double sigmax, double* obj, double* grad,
                                                float* yhat, double* xs, double* gpart,
                                                double* jpart) {
    const int r = blockIdx.x;
    const int q = threadIdx.x & 3, c = threadIdx.x >> 2;
    const size_t NG = (size_t)NT + (size_t)NX * S;
    const double* th = prm + (size_t)r * NG;
    const double* x0 = th + NT;                      // [S][4] initial states of restart r
    const int qc = q < NY ? q : 0;                   // lane 3 has no output row (dy = 0 there)
    double a0[NX], a1[NX], b0[NU], b1[NU], c0[NX], c1[NX], w1[NZ], w2[NH], w2c[NH];
#pragma unroll
    for (int j = 0; j < NX; ++j) {
        a0[j] = th[OA0 + q * NX + j];
        a1[j] = th[OA1 + q * NX + j];
        c0[j] = th[OC0 + qc * NX + j];
        c1[j] = th[OC1 + qc * NX + j];
    }
#pragma unroll
    for (int j = 0; j < NU; ++j) {
        b0[j] = th[OB0 + q * NU + j];
        b1[j] = th[OB1 + q * NU + j];
    }
#pragma unroll
    for (int j = 0; j < NZ; ++j) w1[j] = th[OW1 + q * NZ + j];
#pragma unroll
    for (int j = 0; j < NH; ++j) {
        w2[j] = th[OW2 + q * NH + j];
        w2c[j] = th[OW2 + j * NH + q];               // column q: dh1_q = sum_i W2[i][q] da2_i
    }
    const double bb1 = th[OB_1 + q], bb2 = th[OB_2 + q], w3 = th[OW3 + q], bb3 = th[OB_3];
    const bool want_grad = grad != nullptr;
    const size_t RS = (size_t)R * S;
    const double cc = 2.0 / ((double)K * (double)S);
    for (int s0 = 0; s0 < S; s0 += CH) {
        const bool act = s0 + c < S;
        const int s = act ? s0 + c : S - 1;          // idle chains shadow the last sequence
        const size_t rs = (size_t)r * S + s;
        const float* us = u + (size_t)s * K * NU;
        const float* ys = y ? y + (size_t)s * K * NY : nullptr;
        double xq = x0[(size_t)s * NX + q];
        double J = 0.0;
        // forward sweep; u_k and y_k are loaded one step ahead (their L2 latency would otherwise
        // sit on the chain), the step record (x, h1, h2, y^, p) is kept for the backward sweep
        double un[NU], yn = 0.0;
#pragma unroll
        for (int j = 0; j < NU; ++j) un[j] = K > 0 ? (double)us[j] : 0.0;
        if (ys && q < NY && K > 0) yn = (double)ys[q];
        for (int k = 0; k < K; ++k) {
            double x[NX], uk[NU], h1[NH];
#pragma unroll
            for (int j = 0; j < NU; ++j) uk[j] = un[j];
            const double yk = yn;
            if (k + 1 < K) {
#pragma unroll
                for (int j = 0; j < NU; ++j) un[j] = (double)us[(size_t)(k + 1) * NU + j];
                if (ys && q < NY) yn = (double)ys[(size_t)(k + 1) * NY + q];
            }
#pragma unroll
            for (int j = 0; j < NX; ++j) x[j] = q4get(xq, j);
            // the chain runs x -> eta -> p -> x+; everything affine in p is split as
            // M0 (x, u) + p M1 (x, u), with both halves formed while eta is evaluated, and the
            // dot products are pairwise trees (short dependency chains)
            const double au = fma(w1[NX + 2], uk[2], fma(w1[NX + 1], uk[1], fma(w1[NX], uk[0], bb1)));
            const double a = au + (fma(w1[1], x[1], w1[0] * x[0]) + fma(w1[3], x[3], w1[2] * x[2]));
            const double s0 = (fma(a0[1], x[1], a0[0] * x[0]) + fma(a0[3], x[3], a0[2] * x[2])) +
                              fma(b0[2], uk[2], fma(b0[1], uk[1], b0[0] * uk[0]));
            const double s1 = (fma(a1[1], x[1], a1[0] * x[0]) + fma(a1[3], x[3], a1[2] * x[2])) +
                              fma(b1[2], uk[2], fma(b1[1], uk[1], b1[0] * uk[0]));
            const double t0 = fma(c0[1], x[1], c0[0] * x[0]) + fma(c0[3], x[3], c0[2] * x[2]);
            const double t1 = fma(c1[1], x[1], c1[0] * x[0]) + fma(c1[3], x[3], c1[2] * x[2]);
            const double h1q = tanh_d(a);
#pragma unroll
            for (int j = 0; j < NH; ++j) h1[j] = q4get(h1q, j);
            const double a2 = bb2 + (fma(w2[1], h1[1], w2[0] * h1[0]) + fma(w2[3], h1[3], w2[2] * h1[2]));
            const double h2q = tanh_d(a2);
            const double p = q4sum(w3 * h2q) + bb3;
            const double yq = fma(p, t1, t0);
            const double xn = fma(p, s1, s0);
            if (want_grad && act) {
                double* rec = xs + ((size_t)k * RS + rs) * REC;
                rec[q] = xq;
                rec[NX + q] = h1q;
                rec[2 * NX + q] = h2q;
                rec[3 * NX + q] = yq;
                if (q == 0) rec[4 * NX] = p;
            }
            if (q < NY) {
                if (yhat && act) yhat[(rs * K + k) * NY + q] = (float)yq;
                if (ys) {
                    const double e = yk - yq;
                    J = fma(e, e, J);
                }
            }
            xq = xn;
        }
        J = q4sum(J);
        if (ys && act && q == 0) jpart[rs] = K > 0 ? J / K : 0.0;
        if (!want_grad) continue;
        double ga0[NX] = {}, ga1[NX] = {}, gb0[NU] = {}, gb1[NU] = {}, gc0[NX] = {}, gc1[NX] = {};
        double gw1[NZ] = {}, gw2[NH] = {};
        double gbb1 = 0.0, gbb2 = 0.0, gw3 = 0.0, gbb3 = 0.0;
        double lam[NX] = {0.0, 0.0, 0.0, 0.0};       // dF/dx_{k+1}, every lane holds all of it
        // backward sweep over the stored records; record k-1 is loaded while step k runs, so
        // the chain per step is the adjoint arithmetic alone
        double nx[NX], nh1[NH], nh2 = 0.0, nyq = 0.0, npp = 0.0, nu[NU], ny = 0.0;
        auto load = [&](int k) {
            const double* rec = xs + ((size_t)k * RS + rs) * REC;
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                nx[j] = rec[j];
                nh1[j] = rec[NX + j];
            }
            nh2 = rec[2 * NX + q];
            nyq = rec[3 * NX + q];
            npp = rec[4 * NX];
#pragma unroll
            for (int j = 0; j < NU; ++j) nu[j] = (double)us[(size_t)k * NU + j];
            ny = q < NY ? (double)ys[(size_t)k * NY + q] : 0.0;
        };
        if (K > 0) load(K - 1);
        for (int k = K - 1; k >= 0; --k) {
            double x[NX], uk[NU], h1[NH];
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                x[j] = nx[j];
                h1[j] = nh1[j];
            }
#pragma unroll
            for (int j = 0; j < NU; ++j) uk[j] = nu[j];
            const double h2q = nh2, p = npp, h1q = pick4(h1, q);
            const double dyq = q < NY ? cc * (nyq - ny) : 0.0;
            if (k > 0) load(k - 1);
            const double lq = pick4(lam, q);
            // off the adjoint chain: the record's contractions and the tanh derivatives
            const double al = (fma(a1[1], x[1], a1[0] * x[0]) + fma(a1[3], x[3], a1[2] * x[2])) +
                              fma(b1[2], uk[2], fma(b1[1], uk[1], b1[0] * uk[0]));   // A1 x + B1 u
            const double gm = fma(c1[1], x[1], c1[0] * x[0]) + fma(c1[3], x[3], c1[2] * x[2]);
            const double K2 = w3 * (1.0 - h2q * h2q), K1 = 1.0 - h1q * h1q;
            double sl[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j)
                sl[j] = fma(fma(p, a1[j], a0[j]), lq, fma(p, c1[j], c0[j]) * dyq);
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                const double d = lq * x[j], e = dyq * x[j];
                ga0[j] += d;
                ga1[j] = fma(p, d, ga1[j]);
                gc0[j] += e;
                gc1[j] = fma(p, e, gc1[j]);
            }
#pragma unroll
            for (int j = 0; j < NU; ++j) {
                const double d = lq * uk[j];
                gb0[j] += d;
                gb1[j] = fma(p, d, gb1[j]);
            }
            // the adjoint chain: dp = <A1, lam x^T> + <B1, lam u^T> + <C1, dy x^T>
            const double dp = q4sum(fma(lq, al, dyq * gm));
            gbb3 += dp;
            gw3 = fma(dp, h2q, gw3);
            const double da2q = dp * K2;
            gbb2 += da2q;
#pragma unroll
            for (int j = 0; j < NH; ++j) gw2[j] = fma(da2q, h1[j], gw2[j]);
            const double g0 = q4get(da2q, 0), g1 = q4get(da2q, 1), g2 = q4get(da2q, 2), g3 = q4get(da2q, 3);
            const double da1q = (fma(w2c[1], g1, w2c[0] * g0) + fma(w2c[3], g3, w2c[2] * g2)) * K1;
            gbb1 += da1q;
#pragma unroll
            for (int j = 0; j < NX; ++j) gw1[j] = fma(da1q, x[j], gw1[j]);
#pragma unroll
            for (int j = 0; j < NU; ++j) gw1[NX + j] = fma(da1q, uk[j], gw1[NX + j]);
            // lam_k = A^T lam_{k+1} + C^T dy_k + W1x^T da1: row q's share of every column, summed
#pragma unroll
            for (int j = 0; j < NX; ++j) lam[j] = q4sum(fma(w1[j], da1q, sl[j]));
        }
        if (!act) continue;
        grad[(size_t)r * NG + NT + (size_t)NX * s + q] = fma(sigmax, x0[(size_t)s * NX + q], pick4(lam, q));
        double* gp = gpart + rs * NT;
#pragma unroll
        for (int j = 0; j < NX; ++j) {
            gp[OA0 + q * NX + j] = ga0[j];
            gp[OA1 + q * NX + j] = ga1[j];
            if (q < NY) {
                gp[OC0 + q * NX + j] = gc0[j];
                gp[OC1 + q * NX + j] = gc1[j];
            }
        }
#pragma unroll
        for (int j = 0; j < NU; ++j) {
            gp[OB0 + q * NU + j] = gb0[j];
            gp[OB1 + q * NU + j] = gb1[j];
        }
#pragma unroll
        for (int j = 0; j < NZ; ++j) gp[OW1 + q * NZ + j] = gw1[j];
#pragma unroll
        for (int j = 0; j < NH; ++j) gp[OW2 + q * NH + j] = gw2[j];
        gp[OB_1 + q] = gbb1;
        gp[OB_2 + q] = gbb2;
        gp[OW3 + q] = gw3;
        if (q == 0) gp[OB_3] = gbb3;
    }
    __syncthreads();
    if (want_grad) {
        for (int i = threadIdx.x; i < NT; i += blockDim.x) {
            double acc = 0.0;
            for (int s = 0; s < S; ++s) acc += gpart[((size_t)r * S + s) * NT + i];
            grad[(size_t)r * NG + i] = fma(sigma2, th[i], acc);
        }
    }
    if (obj && threadIdx.x == 0) {
        double Jt = 0.0, t2 = 0.0, x2 = 0.0;
        for (int s = 0; s < S; ++s) Jt += jpart[(size_t)r * S + s];
        for (int i = 0; i < NT; ++i) t2 = fma(th[i], th[i], t2);
        for (size_t i = 0; i < (size_t)S * NX; ++i) x2 = fma(x0[i], x0[i], x2);
        obj[r] = (S > 0 ? Jt / S : 0.0) + 0.5 * sigma2 * t2 + 0.5 * sigmax * x2;
    }
}

// Adam ("a fixed number of Adam gradient-descend steps") on R x n parameters, in place;
// mask[i] = 0 freezes parameter i (the LTI pre-fit of reading LPV2 freezes M1 and eta).
__global__ void k_adam(size_t total, int n, double* w, const double* g, double* m, double* v,
                       double lr, double b1, double b2, double eps, double c1, double c2,
                       const uint8_t* mask) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    if (mask && !mask[i % (size_t)n]) return;
    const double gi = g[i];
    const double mi = fma(b1, m[i], (1.0 - b1) * gi);
    const double vi = fma(b2, v[i], (1.0 - b2) * gi * gi);
    m[i] = mi;
    v[i] = vi;
    w[i] -= lr * (mi * c1) / (sqrt(vi * c2) + eps);
}

}  // namespace lpv

using namespace lpv;

extern "C" {

size_t sph_lpv_scratch_bytes(int R, int S, int K) {
    if (R <= 0 || S <= 0 || K < 0) return 0;
    const size_t RS = (size_t)R * S;
    return sizeof(double) * (RS * (size_t)K * REC + RS * NT + RS);
}

sph_status sph_lpv_eval(int R, int S, int K, const double* params, const float* u, const float* y,
                        double sigma2, double sigmax, double* obj, double* grad, float* yhat,
                        void* scratch, size_t scratch_bytes, void* stream) {
    if (R <= 0 || S <= 0 || K < 0 || !params || (K > 0 && !u)) return SPH_EINVAL;
    if ((obj || grad) && K > 0 && !y) return SPH_EINVAL;
    if (!(sigma2 >= 0.0) || !(sigmax >= 0.0)) return SPH_EINVAL;
    if (!scratch || scratch_bytes < sph_lpv_scratch_bytes(R, S, K)) return SPH_EINVAL;
    if (K == 0 && grad) return SPH_EINVAL;
    const size_t RS = (size_t)R * S;
    double* xs = static_cast<double*>(scratch);
    double* gpart = xs + RS * (size_t)K * REC;
    double* jpart = gpart + RS * NT;
    k_lpv<<<R, LPV_T, 0, static_cast<cudaStream_t>(stream)>>>(R, S, K, params, u, y, sigma2, sigmax,
                                                             obj, grad, yhat, xs, gpart, jpart);
    return cudaGetLastError() == cudaSuccess ? SPH_OK : SPH_ECUDA;
}

sph_status sph_lpv_adam(int R, int n, double* w, const double* g, double* m, double* v, double lr,
                        double beta1, double beta2, double eps, int t, const uint8_t* mask,
                        void* stream) {
    if (R <= 0 || n <= 0 || t < 1 || !w || !g || !m || !v) return SPH_EINVAL;
    if (!(lr > 0.0) || !(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0) || !(eps > 0.0))
        return SPH_EINVAL;
    const size_t total = (size_t)R * n;
    const double c1 = 1.0 / (1.0 - std::pow(beta1, t)), c2 = 1.0 / (1.0 - std::pow(beta2, t));
    k_adam<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        total, n, w, g, m, v, lr, beta1, beta2, eps, c1, c2, mask);
    return cudaGetLastError() == cudaSuccess ? SPH_OK : SPH_ECUDA;
}

}  // extern "C"
