// sph_jac.cuh -- linearization of the continuous-time model.
//
// The paper obtains "linearized dynamics around arbitrary operating points" by automatic
// differentiation of the state-transition function (P:259 item 2) and shows the eigenvalues of
// the linearized open-loop system along trajectories (Figs. 5-6).  Here the Jacobians
// A = df/dx (n_x x n_x) and B = df/du (n_x x 3) of
//   f(x, u) = [vel, a(x), rd, thd, (F_b + u_xy) / m_B, (T_b + tau) / J]
// with x = [pos (N x 2, canonical id order), vel (N x 2), r_x, r_y, theta, rd_x, rd_y, thd],
// n_x = 4N + 6, are computed by forward-mode (tangent-linear, "dual number") differentiation in
// float64: every column of [A | B] is one directional derivative along a unit seed, and the seeds
// are the batch dimension of the kernels (one CTA column per seed), the way the ensemble path
// batches rollouts.  Neighbour sets are the float64 predicates of the oracle (fixed at the
// operating point: f is piecewise smooth and the support boundaries carry zero kernel value and
// gradient).  Tangent rules, with x_ij = x_i - x_j, r = |x_ij|, dr = x_ij . dx_ij / r:
//   d rho_i = m [ sum_j W'(r_ij) dr_ij + gamma1 sum_g W'(r_ig) dr_ig ]        (Eq. density_update)
//   d (P/rho^2)_i = d rho_i (k / rho_i^2 - 2 P_i / rho_i^3)                     (Eq. EOS)
//   a_i^ff = m sum_j s_ij g_ij x_ij,  s = Pi_ij - Q_i - Q_j,  g = W'(r) / r     (Eqs. momentum, viscous)
//   d a_i^ff = m sum_j [ ds g x + s (g'(r) dr x + g dx) ],  g' = (W'' - g) / r
//   G_ig = c_ig gs(r) x_ig, c = sgn 2m^2 Q_i + m^2 beta / rho_i min(v.x, 0) / (r^2 + eps h^2)
//   (Eqs. pressure_b2f, viscous_b2f; gs = W_s3' / r), ghost tangents from Eq. kinematicghost:
//   d x_g = d r + d theta z x arm_g,  d v_g = d rd + d thd z x arm_g - thd d theta arm_g.
#pragma once
#include "sph_device.cuh"

namespace sph {

constexpr int JAC_NCAP = 48;   // fluid neighbours per particle (float64 2h predicate)
constexpr int JAC_GCAP = 48;   // ghosts per particle within 2h (density) / h (forces)
constexpr int JAC_T = 128;     // threads of the dense (body / input seed) column CTA
constexpr int JAC_HCAP = 192;  // particles within two neighbour hops of a particle
constexpr int JAC_PT = 64;     // threads of the sparse (particle seed) column CTA

struct JacParams {
    int N, G, nx;                // particles, ghosts, state dimension 4N + 6
    double h, m, rho0, k, gamma1, alpha2h, beta, eps_h2, sgn2m2, m2, mB, J;
    int clampP;                  // negative pressures clamped to 0 (dP/drho = 0 there)
    double H2, h2;               // (2h)^2, h^2 (float64 predicates, as the oracle)
    double wc, ws;               // w_cb_const, 10 / pi (kernel constants without h powers)
};

struct JacPtrs {
    const double2* pos;          // [N] canonical order
    const double2* vel;          // [N]
    const double* body;          // [6]
    const double2* gB;           // [G] body frame
    double2* gpos;               // [G]
    double2* gvel;               // [G]
    double2* garm;               // [G] x_g - r
    int* nf_cnt;                 // [N]
    int* nf;                     // [N][JAC_NCAP]
    int* g2_cnt;                 // [N]
    int* g2;                     // [N][JAC_GCAP] ghosts within 2h
    int* g1_cnt;                 // [N]
    int* g1;                     // [N][JAC_GCAP] ghosts within h
    double* rho;                 // [N]
    double* P;                   // [N]
    double* Q;                   // [N] P / rho^2
    int* hop_cnt;                // [N]
    int* hop;                    // [N][JAC_HCAP] {k} u NF(k) u NF(NF(k)): rows a seed on k touches
    double* drho;                // [9][N] tangent densities of the body / input seeds
    double* A;                   // [nx][nx] row-major output (zeroed before the seeds run)
    double* B;                   // [nx][3]  row-major output
    double* bpart;               // [9][ceil(N / JAC_T)][3] body partials of the dense columns
    int* overflow;               // [1]
};

// cubic spline (Eq. cubicspline) in r: W, dW/dr, d2W/dr2
__device__ __forceinline__ void jac_wcb(const JacParams& J, double r, double* W1, double* W2) {
    const double q = r / J.h, h3 = J.h * J.h * J.h, h4 = h3 * J.h;
    const double a = 2.0 - q, b = 1.0 - q;
    double w1 = 0.0, w2 = 0.0;
    if (q < 1.0) {
        w1 = -3.0 * a * a + 12.0 * b * b;
        w2 = 6.0 * a - 24.0 * b;
    } else if (q < 2.0) {
        w1 = -3.0 * a * a;
        w2 = 6.0 * a;
    }
    *W1 = J.wc * w1 / h3;
    *W2 = J.wc * w2 / h4;
}

// spiky (Eq. spiky3) in r < h: dW/dr, d2W/dr2
__device__ __forceinline__ void jac_ws(const JacParams& J, double r, double* W1, double* W2) {
    const double h5 = J.h * J.h * J.h * J.h * J.h, e = J.h - r;
    *W1 = r < J.h ? -3.0 * J.ws * e * e / h5 : 0.0;
    *W2 = r < J.h ? 6.0 * J.ws * e / h5 : 0.0;
}

__device__ __forceinline__ double dot2(double2 a, double2 b) { return a.x * b.x + a.y * b.y; }
__device__ __forceinline__ double cross2(double2 a, double2 b) { return a.x * b.y - a.y * b.x; }
__device__ __forceinline__ double2 zx(double2 a) { return make_double2(-a.y, a.x); }   // z x a

// unit seed d: tangent of the fluid position / velocity of particle j and of the body
__device__ __forceinline__ double2 seed_pos(int d, int j) {
    return make_double2(d == 2 * j ? 1.0 : 0.0, d == 2 * j + 1 ? 1.0 : 0.0);
}
__device__ __forceinline__ double2 seed_vel(const JacParams& J, int d, int j) {
    return make_double2(d == 2 * J.N + 2 * j ? 1.0 : 0.0, d == 2 * J.N + 2 * j + 1 ? 1.0 : 0.0);
}
struct BodySeed {
    double2 dr, drd, du;
    double dth, dthd, dtau;
};
__device__ __forceinline__ BodySeed body_seed(const JacParams& J, int d) {
    const int b0 = 4 * J.N;
    BodySeed s;
    s.dr = make_double2(d == b0 ? 1.0 : 0.0, d == b0 + 1 ? 1.0 : 0.0);
    s.dth = d == b0 + 2 ? 1.0 : 0.0;
    s.drd = make_double2(d == b0 + 3 ? 1.0 : 0.0, d == b0 + 4 ? 1.0 : 0.0);
    s.dthd = d == b0 + 5 ? 1.0 : 0.0;
    s.du = make_double2(d == J.nx ? 1.0 : 0.0, d == J.nx + 1 ? 1.0 : 0.0);
    s.dtau = d == J.nx + 2 ? 1.0 : 0.0;
    return s;
}

// entry (row, seed d) of [A | B]
__device__ __forceinline__ void jac_put(const JacParams& J, const JacPtrs& X, int row, int d, double v) {
    if (d < J.nx) X.A[(size_t)row * J.nx + d] = v;
    else X.B[(size_t)row * 3 + (d - J.nx)] = v;
}

// Eq. kinematicghost in float64
__global__ void k_jac_ghosts(JacParams J, JacPtrs X) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= J.G) return;
    const double* b = X.body;
    double s, c;
    sincos(b[2], &s, &c);
    const double2 q = X.gB[g];
    const double2 arm = make_double2(c * q.x - s * q.y, s * q.x + c * q.y);
    X.garm[g] = arm;
    X.gpos[g] = make_double2(arm.x + b[0], arm.y + b[1]);
    X.gvel[g] = make_double2(b[3] - b[5] * arm.y, b[4] + b[5] * arm.x);
}

// float64 neighbour sets (ascending index, as the oracle) + density and EOS at the point.
// One warp per particle: lanes test 32 candidates at a time, ballots keep the ascending order.
__global__ void k_jac_prep(JacParams J, JacPtrs X) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= J.N) return;   // warp-uniform
    const double2 xi = X.pos[i];
    const unsigned below = (1u << lane) - 1u;
    int n = 0, n2 = 0, n1 = 0;
    double ws = 0.0, wg = 0.0;
    const double h2i = 1.0 / (J.h * J.h);
    auto wcb = [&](double r) {
        const double q = r / J.h, a = 2.0 - q, b = 1.0 - q;
        const double w = q < 1.0 ? a * a * a - 4.0 * b * b * b : (q < 2.0 ? a * a * a : 0.0);
        return J.wc * w * h2i;
    };
    for (int j0 = 0; j0 < J.N; j0 += 32) {
        const int j = j0 + lane;
        bool in = false;
        double r2 = 0.0;
        if (j < J.N && j != i) {
            const double2 xj = X.pos[j];
            const double dx = xi.x - xj.x, dy = xi.y - xj.y;
            r2 = dx * dx + dy * dy;
            in = r2 < J.H2;
        }
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (in) {
            const int at = n + __popc(m & below);
            if (at < JAC_NCAP) X.nf[(size_t)i * JAC_NCAP + at] = j;
            ws += wcb(sqrt(r2));
        }
        n += __popc(m);
    }
    for (int g0 = 0; g0 < J.G; g0 += 32) {
        const int g = g0 + lane;
        double r2 = 1e300;
        if (g < J.G) {
            const double2 xg = X.gpos[g];
            const double dx = xi.x - xg.x, dy = xi.y - xg.y;
            r2 = dx * dx + dy * dy;
        }
        const bool in2 = r2 < J.H2, in1 = r2 < J.h2;
        const unsigned m2 = __ballot_sync(0xffffffffu, in2), m1 = __ballot_sync(0xffffffffu, in1);
        if (in2) {
            const int at = n2 + __popc(m2 & below);
            if (at < JAC_GCAP) X.g2[(size_t)i * JAC_GCAP + at] = g;
            wg += wcb(sqrt(r2));
        }
        if (in1) {
            const int at = n1 + __popc(m1 & below);
            if (at < JAC_GCAP) X.g1[(size_t)i * JAC_GCAP + at] = g;
        }
        n2 += __popc(m2);
        n1 += __popc(m1);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        ws += __shfl_xor_sync(0xffffffffu, ws, d);
        wg += __shfl_xor_sync(0xffffffffu, wg, d);
    }
    if (lane == 0) {
        if (n > JAC_NCAP || n2 > JAC_GCAP || n1 > JAC_GCAP) atomicExch(X.overflow, 1);
        X.nf_cnt[i] = min(n, JAC_NCAP);
        X.g2_cnt[i] = min(n2, JAC_GCAP);
        X.g1_cnt[i] = min(n1, JAC_GCAP);
        const double rho = J.m * (wcb(0.0) + ws + J.gamma1 * wg);   // self term
        double P = J.k * (rho - J.rho0);
        if (J.clampP && P < 0.0) P = 0.0;
        X.rho[i] = rho;
        X.P[i] = P;
        X.Q[i] = P / (rho * rho);
    }
}

// Tangent density of particle i along seed d.
__device__ __forceinline__ double jac_drho_i(const JacParams& J, const JacPtrs& X, int d, int i,
                                             const BodySeed& bs) {
    const double2 xi = X.pos[i], dxi = seed_pos(d, i);
    double acc = 0.0, accg = 0.0;
    for (int t = 0; t < X.nf_cnt[i]; ++t) {
        const int j = X.nf[(size_t)i * JAC_NCAP + t];
        const double2 x = make_double2(xi.x - X.pos[j].x, xi.y - X.pos[j].y);
        const double2 sj = seed_pos(d, j);
        const double2 dx = make_double2(dxi.x - sj.x, dxi.y - sj.y);
        const double r = sqrt(dot2(x, x));
        if (r > 0.0) {
            double W1, W2;
            jac_wcb(J, r, &W1, &W2);
            acc += W1 * dot2(x, dx) / r;
        }
    }
    for (int t = 0; t < X.g2_cnt[i]; ++t) {
        const int g = X.g2[(size_t)i * JAC_GCAP + t];
        const double2 xg = X.gpos[g], arm = X.garm[g];
        const double2 x = make_double2(xi.x - xg.x, xi.y - xg.y);
        const double2 dxg = make_double2(bs.dr.x - bs.dth * arm.y, bs.dr.y + bs.dth * arm.x);
        const double2 dx = make_double2(dxi.x - dxg.x, dxi.y - dxg.y);
        const double r = sqrt(dot2(x, x));
        if (r > 0.0) {
            double W1, W2;
            jac_wcb(J, r, &W1, &W2);
            accg += W1 * dot2(x, dx) / r;
        }
    }
    return J.m * (acc + J.gamma1 * accg);
}

// tangent densities: thread (seed d0 + blockIdx.y, particle i)  (dense: body seeds)
__global__ void k_jac_drho(JacParams J, JacPtrs X, int d0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= J.N) return;
    const int d = d0 + blockIdx.y;
    X.drho[(size_t)blockIdx.y * J.N + i] = jac_drho_i(J, X, d, i, body_seed(J, d));
}

// Tangent acceleration of particle i along seed d; drho_of(j) gives the tangent density of j.
// Adds the ghost reactions' tangents to the body force / torque accumulators.
template <class DR>
__device__ __forceinline__ double2 jac_dacc_i(const JacParams& J, const JacPtrs& X, int d, int i,
                                              const BodySeed& bs, double thd, DR&& drho_of,
                                              double& dFx, double& dFy, double& dT) {
    const double2 xi = X.pos[i], vi = X.vel[i];
    const double2 dxi = seed_pos(d, i), dvi = seed_vel(J, d, i);
    const double rhoi = X.rho[i], Qi = X.Q[i], Pi = X.P[i], drhoi = drho_of(i);
    const double ki = (J.clampP && rhoi < J.rho0) ? 0.0 : J.k;   // dP/drho (clamped: 0)
    const double dQi = drhoi * (ki / (rhoi * rhoi) - 2.0 * Pi / (rhoi * rhoi * rhoi));
    double2 da = make_double2(0.0, 0.0);   // d a_i^ff / m
    for (int t = 0; t < X.nf_cnt[i]; ++t) {
        const int j = X.nf[(size_t)i * JAC_NCAP + t];
        const double2 xj = X.pos[j], vj = X.vel[j];
        const double2 x = make_double2(xi.x - xj.x, xi.y - xj.y);
        const double2 v = make_double2(vi.x - vj.x, vi.y - vj.y);
        const double2 sj = seed_pos(d, j), tj = seed_vel(J, d, j);
        const double2 dx = make_double2(dxi.x - sj.x, dxi.y - sj.y);
        const double2 dv = make_double2(dvi.x - tj.x, dvi.y - tj.y);
        const double r2 = dot2(x, x);
        if (!(r2 > 0.0)) continue;
        const double r = sqrt(r2);
        double W1, W2;
        jac_wcb(J, r, &W1, &W2);
        const double g = W1 / r, dg_dr = (W2 - g) / r;
        const double dr = dot2(x, dx) / r;
        const double rhoj = X.rho[j], Qj = X.Q[j], Pj = X.P[j], drhoj = drho_of(j);
        const double kj = (J.clampP && rhoj < J.rho0) ? 0.0 : J.k;
        const double dQj = drhoj * (kj / (rhoj * rhoj) - 2.0 * Pj / (rhoj * rhoj * rhoj));
        const double den = r2 + J.eps_h2, c = dot2(v, x) / den;
        const double rs = rhoi + rhoj;
        const double Pi_ = J.alpha2h * c / rs;
        const double dc = (dot2(dv, x) + dot2(v, dx) - c * 2.0 * dot2(x, dx)) / den;
        const double dPi = J.alpha2h * (dc / rs - c * (drhoi + drhoj) / (rs * rs));
        const double s = Pi_ - Qi - Qj, ds = dPi - dQi - dQj;
        const double dg = dg_dr * dr;
        da.x += ds * g * x.x + s * (dg * x.x + g * dx.x);
        da.y += ds * g * x.y + s * (dg * x.y + g * dx.y);
    }
    da.x *= J.m;
    da.y *= J.m;
    for (int t = 0; t < X.g1_cnt[i]; ++t) {   // fluid-ghost forces (spiky, support h)
        const int gi = X.g1[(size_t)i * JAC_GCAP + t];
        const double2 xg = X.gpos[gi], vg = X.gvel[gi], arm = X.garm[gi];
        const double2 x = make_double2(xi.x - xg.x, xi.y - xg.y);
        const double2 v = make_double2(vi.x - vg.x, vi.y - vg.y);
        const double2 dxg = make_double2(bs.dr.x - bs.dth * arm.y, bs.dr.y + bs.dth * arm.x);
        const double2 dvg = make_double2(bs.drd.x - bs.dthd * arm.y - thd * bs.dth * arm.x,
                                         bs.drd.y + bs.dthd * arm.x - thd * bs.dth * arm.y);
        const double2 dx = make_double2(dxi.x - dxg.x, dxi.y - dxg.y);
        const double2 dv = make_double2(dvi.x - dvg.x, dvi.y - dvg.y);
        const double r2 = dot2(x, x);
        if (!(r2 > 0.0)) continue;
        const double r = sqrt(r2);
        double W1, W2;
        jac_ws(J, r, &W1, &W2);
        const double gs = W1 / r, dgs = (W2 - gs) / r * (dot2(x, dx) / r);
        const double den = r2 + J.eps_h2, vr = dot2(v, x);
        const double mu = fmin(vr, 0.0);
        const double dmu = vr < 0.0 ? dot2(dv, x) + dot2(v, dx) : 0.0;
        const double cf = J.sgn2m2 * Qi + J.m2 * J.beta / rhoi * mu / den;
        const double dcf = J.sgn2m2 * dQi +
                           J.m2 * J.beta * (-drhoi / (rhoi * rhoi) * mu / den +
                                            (dmu / den - mu * 2.0 * dot2(x, dx) / (den * den)) / rhoi);
        const double2 G = make_double2(cf * gs * x.x, cf * gs * x.y);
        const double2 dG = make_double2(dcf * gs * x.x + cf * (dgs * x.x + gs * dx.x),
                                        dcf * gs * x.y + cf * (dgs * x.y + gs * dx.y));
        da.x += dG.x / J.m;
        da.y += dG.y / J.m;
        dFx -= dG.x;
        dFy -= dG.y;
        // T = sum arm x (-G):  dT = d arm x (-G) + arm x (-dG),  d arm = d theta z x arm
        dT += cross2(make_double2(-bs.dth * arm.y, bs.dth * arm.x), make_double2(-G.x, -G.y)) +
              cross2(arm, make_double2(-dG.x, -dG.y));
    }
    return da;
}

// fixed-order tree over NT threads (deterministic), then the six body rows of the column
template <int NT>
__device__ __forceinline__ void jac_body_rows(const JacParams& J, const JacPtrs& X, int d,
                                              const BodySeed& bs, double dFx, double dFy, double dT,
                                              double (*red)[NT]) {
    red[0][threadIdx.x] = dFx;
    red[1][threadIdx.x] = dFy;
    red[2][threadIdx.x] = dT;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int b = 4 * J.N;
        jac_put(J, X, b + 0, d, bs.drd.x);                  // d r / dt = rd
        jac_put(J, X, b + 1, d, bs.drd.y);
        jac_put(J, X, b + 2, d, bs.dthd);                   // d theta / dt = thd
        jac_put(J, X, b + 3, d, (red[0][0] + bs.du.x) / J.mB);   // (F_b + u) / m_B
        jac_put(J, X, b + 4, d, (red[1][0] + bs.du.y) / J.mB);
        jac_put(J, X, b + 5, d, (red[2][0] + bs.dtau) / J.J);    // (T_b + tau) / J
    }
}

// Dense columns (body / input seeds: every particle may respond): CTA (x, y) handles particles
// [x JAC_T, (x + 1) JAC_T) of seed d0 + y and stores its body partial (fixed-order block tree);
// k_jac_body sums the partials of each seed in block order and writes the six body rows.
__global__ void __launch_bounds__(JAC_T) k_jac_col(JacParams J, JacPtrs X, int d0) {
    __shared__ double red[3][JAC_T];
    const int dl = blockIdx.y, d = d0 + dl;
    const BodySeed bs = body_seed(J, d);
    const double* drho = X.drho + (size_t)dl * J.N;
    const double thd = X.body[5];
    double dFx = 0.0, dFy = 0.0, dT = 0.0;
    const int i = blockIdx.x * JAC_T + threadIdx.x;
    if (i < J.N) {   // (d pos / dt = vel rows are zero for body / input seeds)
        const double2 da = jac_dacc_i(J, X, d, i, bs, thd, [&](int j) { return drho[j]; }, dFx, dFy, dT);
        jac_put(J, X, 2 * J.N + 2 * i, d, da.x);       // d vel / dt = a
        jac_put(J, X, 2 * J.N + 2 * i + 1, d, da.y);
    }
    red[0][threadIdx.x] = dFx;
    red[1][threadIdx.x] = dFy;
    red[2][threadIdx.x] = dT;
    __syncthreads();
    for (int w = JAC_T / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 3) X.bpart[((size_t)dl * gridDim.x + blockIdx.x) * 3 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void k_jac_body(JacParams J, JacPtrs X, int d0, int nblk) {
    const int dl = blockIdx.x, d = d0 + dl;
    if (threadIdx.x != 0) return;
    const BodySeed bs = body_seed(J, d);
    double F[3] = {0.0, 0.0, 0.0};
    for (int b = 0; b < nblk; ++b)
        for (int c = 0; c < 3; ++c) F[c] += X.bpart[((size_t)dl * nblk + b) * 3 + c];
    const int b = 4 * J.N;
    jac_put(J, X, b + 0, d, bs.drd.x);
    jac_put(J, X, b + 1, d, bs.drd.y);
    jac_put(J, X, b + 2, d, bs.dthd);
    jac_put(J, X, b + 3, d, (F[0] + bs.du.x) / J.mB);
    jac_put(J, X, b + 4, d, (F[1] + bs.du.y) / J.mB);
    jac_put(J, X, b + 5, d, (F[2] + bs.dtau) / J.J);
}

// two-hop row sets: H(k) = {k} u NF(k) u NF(NF(k)) (no duplicates).  One warp per particle:
// candidates gathered into shared memory, duplicates dropped in parallel, kept ones compacted.
constexpr int JAC_HOPS_WARPS = 4;
constexpr int JAC_CAND = 1 + JAC_NCAP + JAC_NCAP * JAC_NCAP;
__global__ void __launch_bounds__(32 * JAC_HOPS_WARPS) k_jac_hops(JacParams J, JacPtrs X) {
    extern __shared__ int cand_all[];   // [JAC_HOPS_WARPS][JAC_CAND]
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = blockIdx.x * JAC_HOPS_WARPS + w;
    if (k >= J.N) return;   // warp-uniform
    int* cand = cand_all + w * JAC_CAND;
    const int nk = X.nf_cnt[k];
    if (lane == 0) cand[0] = k;
    for (int t = lane; t < nk; t += 32) cand[1 + t] = X.nf[(size_t)k * JAC_NCAP + t];
    int n = 1 + nk;
    for (int a = 0; a < nk; ++a) {
        const int j = X.nf[(size_t)k * JAC_NCAP + a], nj = X.nf_cnt[j];
        for (int t = lane; t < nj; t += 32) cand[n + t] = X.nf[(size_t)j * JAC_NCAP + t];
        n += nj;
    }
    __syncwarp();
    const unsigned below = (1u << lane) - 1u;
    int kept = 0;
    for (int t0 = 0; t0 < n; t0 += 32) {
        const int t = t0 + lane;
        bool keep = false;
        if (t < n) {
            const int c = cand[t];
            keep = true;
            for (int u = 0; u < t && keep; ++u) keep = cand[u] != c;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int at = kept + __popc(m & below);
            if (at < JAC_HCAP) X.hop[(size_t)k * JAC_HCAP + at] = cand[t];
        }
        kept += __popc(m);
    }
    if (lane == 0) {
        if (kept > JAC_HCAP) atomicExch(X.overflow, 1);
        X.hop_cnt[k] = min(kept, JAC_HCAP);
    }
}

// Sparse column of a particle seed (d < 4N, particle k): the tangent densities live on
// S1 = {k} u NF(k) only (shared memory), the tangent accelerations on H(k) only; every other
// row of the column stays zero (the column is cleared before).  The ghost reactions of the
// wall particles in H(k) feed the body rows.
__global__ void __launch_bounds__(JAC_PT) k_jac_pseed(JacParams J, JacPtrs X, int d0) {
    __shared__ int s1[JAC_NCAP + 1];
    __shared__ double sdr[JAC_NCAP + 1];
    __shared__ double red[3][JAC_PT];
    const int dl = blockIdx.x, d = d0 + dl;
    const bool vseed = d >= 2 * J.N;
    const int k = (vseed ? d - 2 * J.N : d) >> 1;
    const BodySeed bs = body_seed(J, d);    // all zero for particle seeds
    const int n1 = 1 + X.nf_cnt[k];
    for (int t = threadIdx.x; t < n1; t += JAC_PT) {
        const int i = t == 0 ? k : X.nf[(size_t)k * JAC_NCAP + t - 1];
        s1[t] = i;
        sdr[t] = vseed ? 0.0 : jac_drho_i(J, X, d, i, bs);
    }
    __syncthreads();
    auto drho_of = [&](int j) {
        for (int t = 0; t < n1; ++t)
            if (s1[t] == j) return sdr[t];
        return 0.0;
    };
    const double thd = X.body[5];
    double dFx = 0.0, dFy = 0.0, dT = 0.0;
    const int nh = X.hop_cnt[k];
    for (int t = threadIdx.x; t < nh; t += JAC_PT) {
        const int i = X.hop[(size_t)k * JAC_HCAP + t];
        const double2 da = jac_dacc_i(J, X, d, i, bs, thd, drho_of, dFx, dFy, dT);
        X.A[(size_t)(2 * J.N + 2 * i) * J.nx + d] = da.x;
        X.A[(size_t)(2 * J.N + 2 * i + 1) * J.nx + d] = da.y;
    }
    if (vseed && threadIdx.x == 0) X.A[(size_t)(d - 2 * J.N) * J.nx + d] = 1.0;   // d pos_k/dt = vel_k
    jac_body_rows<JAC_PT>(J, X, d, bs, dFx, dFy, dT, red);
}

// canonical-order float64 operating point of rollout b: pos / vel from the float32 state
__global__ void k_jac_import(DevParams P, DevPtrs D, int b, double2* pos, double2* vel, double* body) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const RolloutState* rs = D.rs + b;
    if (s < P.N) {
        const size_t o = (size_t)b * P.N;
        const float4 v = D.pv[rs->sp][o + s];
        const uint32_t id = D.id[rs->ip][o + s];
        pos[id] = make_double2((double)v.x, (double)v.y);
        vel[id] = make_double2((double)v.z, (double)v.w);
    }
    if (s < 6) body[s] = D.body[(size_t)b * 6 + s];
}

}  // namespace sph
