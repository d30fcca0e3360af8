// Calibration utilities: the analytic estimate of the wall correcting factor
// gamma1, Eq. gamma1, on the current state of one rollout.
//   gamma1_i = (rho_i / m_i - sum_f W_i,f) / sum_g W_i,g
// with rho_i := the caller's target density and the printed denominator subscript i_b read as
// the ghost sum (reading G1).  The sums are those of Eq. density_update
// with the canonical float32 support predicate (reading A19), every fluid particle and every
// ghost tested (brute force over shared-memory tiles: a one-off utility, O(N^2) per call).
#pragma once

#include "sph_device.cuh"

namespace sph {

constexpr int G1_T = 256;

// One thread per slot of rollout b; writes, in canonical id order, parts[id] = (sf, sg) in units
// of C/h^2 (sf includes the self term) and g1[id] = gamma1_i (NaN where sg = 0).
__global__ void __launch_bounds__(G1_T) k_gamma1_parts(DevParams P, DevPtrs D, int b, float rt,
                                                       float2* parts, float* g1) {
    __shared__ float2 tile[G1_T];
    const RolloutState* rs = D.rs + b;
    const size_t o = (size_t)b * P.N;
    const float4* pv = D.pv[rs->sp] + o;
    const int i = blockIdx.x * G1_T + threadIdx.x;
    float2 xi = make_float2(0.0f, 0.0f);
    if (i < P.N) {
        const float4 v = pv[i];
        xi = make_float2(v.x, v.y);
    }
    float sf = 0.0f;   // j = i passes the predicate with r = 0: the self term W(0)
    for (int t0 = 0; t0 < P.N; t0 += G1_T) {
        __syncthreads();
        if (t0 + threadIdx.x < P.N) {
            const float4 v = pv[t0 + threadIdx.x];
            tile[threadIdx.x] = make_float2(v.x, v.y);
        }
        __syncthreads();
        const int m = min(G1_T, P.N - t0);
        for (int j = 0; j < m; ++j) {
            const float2 xj = tile[j];
            const float dx = __fsub_rn(xi.x, xj.x), dy = __fsub_rn(xi.y, xj.y);
            const float r2 = dist2(dx, dy);
            if (r2 < P.H2) sf += wcb_poly(r2 > 0.0f ? r2 * rsqrtf(r2) * P.inv_h : 0.0f);
        }
    }
    if (i >= P.N) return;
    // ghosts: hi part for the predicate, hi + lo for the distance (reading B2), as in the
    // density kernel's wall term
    float sg = 0.0f;
    const float4* gst = D.gst + (size_t)b * P.G;
    const float2* glo = D.glo + (size_t)b * P.G;
    for (int g = 0; g < P.G; ++g) {
        const float4 xg = gst[g];
        const float dx = __fsub_rn(xi.x, xg.x), dy = __fsub_rn(xi.y, xg.y);
        if (dist2(dx, dy) < P.H2) {
            const float2 lo = glo[g];
            const float ex = dx - lo.x, ey = dy - lo.y;
            const float r2 = ex * ex + ey * ey;
            sg += wcb_poly(r2 > 0.0f ? r2 * rsqrtf(r2) * P.inv_h : 0.0f);
        }
    }
    const uint32_t id = D.id[rs->ip][o + i];
    parts[id] = make_float2(sf, sg);
    g1[id] = sg > 0.0f ? (rt - sf) / sg : __int_as_float(0x7fc00000);
}

// Wall-layer value: sum of the numerators over the sum of the denominators of the particles
// with sg > 0 (reading G1), in float64, fixed order (thread-strided sums, then a tree).
__global__ void __launch_bounds__(1024) k_gamma1_wall(int n, const float2* parts, float rt,
                                                      double* out) {
    __shared__ double sn[1024], sd[1024];
    double num = 0.0, den = 0.0;
    for (int i = threadIdx.x; i < n; i += 1024) {
        const float2 p = parts[i];
        if (p.y > 0.0f) {
            num += (double)rt - (double)p.x;
            den += (double)p.y;
        }
    }
    sn[threadIdx.x] = num;
    sd[threadIdx.x] = den;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            sn[threadIdx.x] += sn[threadIdx.x + s];
            sd[threadIdx.x] += sd[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sn[0];
        out[1] = sd[0];
    }
}

}  // namespace sph
