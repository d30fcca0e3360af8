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
constexpr int JAC_T = 128;     // threads of the per-seed column CTA

struct JacParams {
    int N, G, nx;                // particles, ghosts, state dimension 4N + 6
    double h, m, rho0, k, gamma1, alpha2h, beta, eps_h2, sgn2m2, m2, mB, J;
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
    double* drho;                // [Dc][N] tangent densities of the current seed chunk
    double* At;                  // [Dc][nx] columns of A (and B) of the current chunk
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

// float64 neighbour sets (ascending index, as the oracle) + density and EOS at the point
__global__ void k_jac_prep(JacParams J, JacPtrs X) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= J.N) return;
    const double2 xi = X.pos[i];
    int n = 0, n2 = 0, n1 = 0;
    double ws = 0.0, wg = 0.0;
    const double h2i = 1.0 / (J.h * J.h);
    auto wcb = [&](double r) {
        const double q = r / J.h, a = 2.0 - q, b = 1.0 - q;
        const double w = q < 1.0 ? a * a * a - 4.0 * b * b * b : (q < 2.0 ? a * a * a : 0.0);
        return J.wc * w * h2i;
    };
    for (int j = 0; j < J.N; ++j) {
        if (j == i) continue;
        const double2 xj = X.pos[j];
        const double dx = xi.x - xj.x, dy = xi.y - xj.y, r2 = dx * dx + dy * dy;
        if (r2 < J.H2) {
            if (n < JAC_NCAP) X.nf[(size_t)i * JAC_NCAP + n] = j;
            ++n;
            ws += wcb(sqrt(r2));
        }
    }
    for (int g = 0; g < J.G; ++g) {
        const double2 xg = X.gpos[g];
        const double dx = xi.x - xg.x, dy = xi.y - xg.y, r2 = dx * dx + dy * dy;
        if (r2 < J.H2) {
            if (n2 < JAC_GCAP) X.g2[(size_t)i * JAC_GCAP + n2] = g;
            ++n2;
            wg += wcb(sqrt(r2));
        }
        if (r2 < J.h2) {
            if (n1 < JAC_GCAP) X.g1[(size_t)i * JAC_GCAP + n1] = g;
            ++n1;
        }
    }
    if (n > JAC_NCAP || n2 > JAC_GCAP || n1 > JAC_GCAP) atomicExch(X.overflow, 1);
    X.nf_cnt[i] = min(n, JAC_NCAP);
    X.g2_cnt[i] = min(n2, JAC_GCAP);
    X.g1_cnt[i] = min(n1, JAC_GCAP);
    const double rho = J.m * (wcb(0.0) + ws + J.gamma1 * wg);   // self term
    const double P = J.k * (rho - J.rho0);
    X.rho[i] = rho;
    X.P[i] = P;
    X.Q[i] = P / (rho * rho);
}

// tangent densities: thread (seed d0 + blockIdx.y, particle i)
__global__ void k_jac_drho(JacParams J, JacPtrs X, int d0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= J.N) return;
    const int d = d0 + blockIdx.y;
    const BodySeed bs = body_seed(J, d);
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
    X.drho[(size_t)blockIdx.y * J.N + i] = J.m * (acc + J.gamma1 * accg);
}

// one CTA per seed d: column d of [A | B] (fluid rows, body rows with a fixed-order reduction)
__global__ void __launch_bounds__(JAC_T) k_jac_col(JacParams J, JacPtrs X, int d0) {
    __shared__ double red[3][JAC_T];
    const int dl = blockIdx.x, d = d0 + dl;
    const BodySeed bs = body_seed(J, d);
    const double* drho = X.drho + (size_t)dl * J.N;
    double* col = X.At + (size_t)dl * J.nx;
    const double thd = X.body[5];
    double dFx = 0.0, dFy = 0.0, dT = 0.0;
    for (int i = threadIdx.x; i < J.N; i += JAC_T) {
        const double2 xi = X.pos[i], vi = X.vel[i];
        const double2 dxi = seed_pos(d, i), dvi = seed_vel(J, d, i);
        const double rhoi = X.rho[i], Qi = X.Q[i], Pi = X.P[i], drhoi = drho[i];
        const double dQi = drhoi * (J.k / (rhoi * rhoi) - 2.0 * Pi / (rhoi * rhoi * rhoi));
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
            const double rhoj = X.rho[j], Qj = X.Q[j], Pj = X.P[j], drhoj = drho[j];
            const double dQj = drhoj * (J.k / (rhoj * rhoj) - 2.0 * Pj / (rhoj * rhoj * rhoj));
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
        col[2 * i] = dvi.x;                     // d pos / dt = vel
        col[2 * i + 1] = dvi.y;
        col[2 * J.N + 2 * i] = da.x;            // d vel / dt = a
        col[2 * J.N + 2 * i + 1] = da.y;
    }
    red[0][threadIdx.x] = dFx;
    red[1][threadIdx.x] = dFy;
    red[2][threadIdx.x] = dT;
    __syncthreads();
    for (int w = JAC_T / 2; w > 0; w >>= 1) {   // fixed-order tree: deterministic
        if (threadIdx.x < w)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* b = col + 4 * J.N;
        b[0] = bs.drd.x;                        // d r / dt = rd
        b[1] = bs.drd.y;
        b[2] = bs.dthd;                         // d theta / dt = thd
        b[3] = (red[0][0] + bs.du.x) / J.mB;    // (F_b + u) / m_B
        b[4] = (red[1][0] + bs.du.y) / J.mB;
        b[5] = (red[2][0] + bs.dtau) / J.J;     // (T_b + tau) / J
    }
}

// A[r][d0 + c] = At[c][r] for the chunk's seeds c < nxc (the state seeds), tiled transpose;
// B[r][k] = At[nx + k - d0][r] for the input seeds in the chunk.
__global__ void k_jac_store(JacParams J, const double* __restrict__ At, int d0, int dc,
                            double* __restrict__ A, double* __restrict__ B) {
    __shared__ double tile[32][33];
    const int cb = blockIdx.x * 32, rb = blockIdx.y * 32;   // seed (column) block, row block
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = cb + k, r = rb + threadIdx.x;
        tile[k][threadIdx.x] = (c < dc && r < J.nx) ? At[(size_t)c * J.nx + r] : 0.0;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = rb + k, c = cb + threadIdx.x;
        if (r >= J.nx || c >= dc) continue;
        const int d = d0 + c;
        const double v = tile[threadIdx.x][k];
        if (d < J.nx) A[(size_t)r * J.nx + d] = v;
        else B[(size_t)r * 3 + (d - J.nx)] = v;
    }
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
