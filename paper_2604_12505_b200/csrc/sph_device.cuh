// sph_device.cuh -- device-side data layout, parameters and helpers of the B200-native SPH
// fuel-sloshing step (sm_100a).  P:n = line n of the paper text.
//
// One substep of one rollout is (Algorithm 1, + symplectic Euler):
//   [rebuild, only when needed]
//     k_hash -> k_scan_reduce -> k_scan_tiles -> k_scan_down -> k_scatter -> k_cellsort
//     -> k_gather  (counting sort of the particles by cell, row-major cells of side 2h+skin)
//     -> k_nlist   (per-particle candidate list within 2h+skin from the 3x3 cell block)
//   k_density  Eq. density_update + Eq. EOS over the list
//   k_force    Eqs. momentum, viscous, pressure_b2f / viscous_b2f,
//              Alg. 1 l.8, kick-then-drift of the fluid, per-CTA body partials
//   k_body     Eq. tankdynamics fixed-order fp64 reduction, body kick-drift,
//              Eq. kinematicghost for the next substep, status, rebuild policy
// The neighbour SETS are fixed by the exact float32 predicate |x_i - x_j|^2 < (2h + skin)^2
// (reading A19) when the lists are built; inside k_density / k_force the sums are cut at 2h by
// the kernels' shape (W and dW vanish there, B3), so with the Verlet skin the sums
// equal those of a fresh all-pairs search every substep.
// Every rollout owns whole CTAs (blockIdx.y = rollout): results never depend on the batch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sph {

constexpr int TILE = 256;        // particles (threads) per CTA in the particle kernels
constexpr int SCAN_T = 256;      // threads per scan CTA
constexpr int SCAN_V = 8;        // counts per scan thread
constexpr int SCAN_TILE = SCAN_T * SCAN_V;
constexpr int BODY_T = 128;      // threads of the per-rollout body kernel
constexpr int SORT_LOCAL = 16;   // cells up to this size are sorted in registers
constexpr int KMAX = 24;         // neighbour-list capacity; more -> cell-scan fallback
constexpr int KQ = KMAX / 4;     // the list is stored as quads of int16 offsets (8 B loads)
constexpr int NL_OVERFLOW = 255; // ncnt value marking a particle that uses the fallback
constexpr int DBG_CAP = 64;

struct DevParams {
    int N, G, B;            // fluid particles / ghosts per rollout, rollouts
    int nx, ncell;          // square cell grid: nx * nx cells per rollout
    int ntile, nscan;       // CTAs per rollout (particle kernels, scan kernels)
    int npart;              // per-warp body partials per rollout = ntile * TILE / 32
    int ghost_K, ghost_K1, ghost_full;   // ghost windows for support 2h (density) and h (force)
    float C, inv_C, half;   // cell side (2h + skin), 1/C, half extent of the grid
    float h, inv_h, H2, h2; // h, 1/h, (2h)^2, h^2 in float32 (predicates, reading A19)
    double h2d;             // 2h in double (list radius 2h + skin, rounded once to float)
    float skin0;            // Verlet skin at init (reading B4); adaptive between skin0 and
    float skin_max;         // skin_max when skin_max > skin0 (B5), cells are 2h + skin_max wide
    int perpart;            // 1: per-particle half-skins instead (B6): pair (i, j) is listed within
                            //    2h + hs_i + hs_j, rebuild when some |d_i| reaches 0.98 hs_i
    float Hf;               // fl(2h)
    float hs_min, hs_max;   // B6: half-skin bounds (skin / 2, skin_max / 2)
    float hs_k;             // B6: hs_i = clamp(hs_k |v_i - v_body|, hs_min, hs_max), hs_k = 20 dt
    float mass, m2, rho0, k, gamma1;
    float alpha2h, beta, eps_h2;
    float wcb, dwcb, dws3;  // C/h^2, C/h^3, -30/(pi h^5)
    float mdwcb3, inv_mass; // m * 3C/h^3 (force sums are in units of 3C/h^3), 1/m
    float gsign2m2;         // ghost_pressure_sign * 2 m^2
    float gx, gy, dt;
    float wall_r2;          // particles with |x - r|^2 <= wall_r2 see no ghost within 2h
    float wall1_r2;         // ... no ghost within h
    float ghost_scale;      // G / (2 pi)
    int rebin_every;
    int NA;                 // aux row stride per rollout = N rounded up to even (16-B rows)
    int td, tf, tn;         // slots (threads) per CTA of k_density / k_force / k_nlist_density
    int snake;              // k_force walks the rollouts last to first (L2 reuse after k_density)
    int bsplit;             // body reduction: 1 = k_body sums the npart partials itself;
                            // > 1 = k_body_reduce first sums bsplit fixed chunks (large tanks;
                            // chosen from N only, so bits never depend on B)
    int pf_d, pf_f;         // L2 prefetch distance in CTAs (k_density / k_force; 0 = off)
    int clampP;             // 1: negative pressures clamped to 0 (ablation E1)
    int own_lo, own_n;      // domain decomposition: the particle kernels compute
                            // slots [own_lo, own_lo + own_n) only (default: all N)
    double dtd, m_body, J_body;
};

struct RolloutState {
    int sp;              // particle state buffer parity
    int ip;              // id buffer parity
    int need_rebin;      // rebuild cell list + neighbour lists at the start of the next substep
    int status;          // 0 ok, 1 non-finite, 2 |x| > 1e9, 3 left the grid (sticky)
    int frozen;          // set by k_body at the end of the substep in which status became
                         // non-zero; kernels skip frozen rollouts (the failing substep is
                         // committed whole, so the exported state stays consistent)
    int rebuilds;        // number of rebuilds (diagnostics)
    long long step;      // substeps taken
    long long bad_step;
    int bad_particle;
    float disp;          // bound on any particle's displacement relative to the body
                         // translation since the last rebuild
    int span;            // max |j - i| over all neighbour-list entries (staging window)
    float rbx, rby;      // body position (float) at the last rebuild
    float skin;          // Verlet skin of the current lists (B5: adapted at every rebuild)
    float rl2;           // list radius^2 = fl(2h + skin)^2 (float32 predicate, reading A19)
    float rdisp;         // rebuild when the displacement bound reaches 0.49 skin (< skin / 2)
    long long last_reb;  // substep index of the last rebuild
};

// Verlet skin -> list radius^2 and rebuild threshold (the same float arithmetic everywhere)
__device__ __forceinline__ void skin_set(const DevParams& P, float skin, float* rl2, float* rdisp) {
    const float RL = (float)(P.h2d + (double)skin);
    *rl2 = __fmul_rn(RL, RL);
    *rdisp = (float)(0.49 * (double)skin);
}
// Adaptive skin (B5): at a rebuild that follows I substeps of the old lists, scale the
// skin by sqrt(SKIN_TARGET / I) (a displacement bound that tripped after I substeps needs skin x
// TARGET / I to last TARGET substeps; the square root damps the response), within
// [skin0, skin_max].  A function of the rollout's own history only (batch-invariant bits).
constexpr int SKIN_TARGET = 8;
__device__ __forceinline__ float skin_adapt(const DevParams& P, float skin, long long I) {
    if (!(P.skin_max > P.skin0) || P.perpart) return skin;
    const double s = (double)skin * sqrt((double)SKIN_TARGET / (double)(I > 1 ? I : 1));
    return (float)fmin(fmax(s, (double)P.skin0), (double)P.skin_max);
}

struct Geom {            // float copy of the body state used by the particle kernels
    float rx, ry, th;    // th = theta + angle of ghost 0 (ghost-ring lookup)
    float vx, vy;        // body velocity (relative-displacement bound)
    float pad[3];
};

// Per-particle half-skin (B6), set at every rebuild from the particle's speed relative
// to the body translation: the skin it needs to last ~28 substeps, within [hs_min, hs_max]
// (HS_TARGET sweeps on C4: 10 / 20 / 40 substeps -> 10.0 / 10.45 / 10.3 G/s; on the final
// round-2 build 15 / 20 / 24 / 28 / 34 -> 10.82 / 11.01 / 11.03 / 11.07 / 11.01 G/s).  For
// a large tank whose wall layer moves 10-50x faster than the bulk (C4), a uniform skin sized for
// the wall makes every list long; a per-particle one keeps the bulk's lists short.
constexpr int HS_TARGET = 28;
// (Measured alternative, not kept: raising the floor per rollout with the B5 rule pushes every
// particle's skin up to outlast the few that trip early -- C4 8.5 vs 9.6 G/s.)
__device__ __forceinline__ float half_skin(const DevParams& P, float4 x, const Geom& gm) {
    const float vx = x.z - gm.vx, vy = x.w - gm.vy;
    return fminf(fmaxf(P.hs_k * sqrtf(vx * vx + vy * vy), P.hs_min), P.hs_max);
}

struct DevPtrs {
    float4* pv[2];       // [B][N] sorted-by-cell particle state (x, y, vx, vy), double buffered
    uint32_t* id[2];     // [B][N] canonical id of each slot
    float2* aux;         // [B][N] (rho, P / rho^2)
    uint32_t* skey;      // [B][N] cell of each slot at the last rebuild
    float2* xb;          // [B][N] position of each slot at the last rebuild (Verlet criterion)
    float* hs;           // [B][N] half-skin of each slot (B6; per-particle skin mode only)
    uint2* nbr;          // [B][KQ][N] neighbour candidates: 4 int16 slot offsets j - i per uint2
    uint8_t* ncnt;       // [B][N] list length (NL_OVERFLOW: scan the cells instead)
    uint32_t* key;       // [B][N] rebuild scratch: cell of each (unsorted) slot
    uint32_t* rank;      // [B][N] rebuild scratch: rank inside the cell
    uint32_t* perm;      // [B][N] rebuild scratch: new slot -> old slot
    uint32_t* counts;    // [B][ncell] cell populations (kept zero between rebuilds)
    uint32_t* cstart;    // [B][ncell + 1] exclusive prefix of counts (cell start table)
    uint32_t* tsum;      // [B][nscan] scan tile sums
    float4* gst;         // [B][G] ghost world state (x_hi, y_hi, vx, vy); x_hi = float(x)
    float2* glo;         // [B][G] x - x_hi, y - y_hi (hi/lo pair: the hi part defines the
                         // float32 neighbour predicate, hi + lo feeds the wall force)
    float2* garm;        // [B][G] ghost arm r_g - r (world frame)
    double2* ghost_b;    // [G] body-frame ghost positions
    double* body;        // [B][6] r_x r_y theta rd_x rd_y thd
    double2* body_cs;    // [B] (cos theta, sin theta) of the current body state (k_ghosts)
    float* u_cur;        // [B][3] current ZOH input
    double4* part;       // [B][npart] per-warp (F_x, F_y, T, max relative speed) partials
    double4* part2;      // [B][bsplit] chunk sums of part (bsplit > 1)
    RolloutState* rs;    // [B]
    Geom* geom;          // [B]
    float4* xfer;        // [N] canonical-order export / import staging
    float* xrho;         // [N]
    int* rlist;          // [B] rollouts that rebuild this substep (k_rebuild_plan)
    int* rcount;         // [1] their number
    int* dbg_cnt;        // [3][N] debug neighbour counts
    int* dbg_idx;        // [3][N][DBG_CAP] debug neighbour ids
};

// ---------------------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk global -> shared, completion on an mbarrier)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
// bytes and both addresses must be multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Programmatic dependent launch (the substep chain on the main stream): a kernel waits for its
// predecessor's completion (and memory) before reading anything it produced, and lets its own
// dependents start launching right away, so kernel launch and prologue overlap the tail of the
// previous kernel.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// L2 prefetch of a global range (address and size multiples of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// ---------------------------------------------------------------------------------------
// Small device helpers
// ---------------------------------------------------------------------------------------
// Canonical float32 cell coordinate (reading A19): floor((x - o) * inv), IEEE RN, no FMA.
__device__ __forceinline__ int cell_coord(float x, float o, float inv) {
    return __float2int_rd(__fmul_rn(__fsub_rn(x, o), inv));
}

// Canonical float32 squared distance (reading A19): dx*dx + dy*dy, no contraction.
__device__ __forceinline__ float dist2(float dx, float dy) {
    return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

// Cubic spline (Eq. cubicspline) without its constant C/h^2; q = r/h < 2.
// (2-q)^3 - 4(1-q)^3 expanded = 4 - 6q^2 + 3q^3 (q < 1); (2-q)^3 (1 <= q < 2).
__device__ __forceinline__ float wcb_poly(float q) {
    const float a = 2.0f - q;
    const float inner = fmaf(q * q, fmaf(3.0f, q, -6.0f), 4.0f);
    const float outer = a * a * a;
    return q < 1.0f ? inner : outer;
}

// dW/dq of the cubic spline without C/h^3.
__device__ __forceinline__ float dwcb_poly(float q) {
    float a = 2.0f - q, b = 1.0f - q;
    float d = -3.0f * a * a;
    if (q < 1.0f) d += 12.0f * b * b;
    return d;
}

// Opaque copy of a pointer: stops the compiler from re-deriving it from (rollout, slot) index
// arithmetic inside the neighbour loops, so a neighbour address is one IMAD.WIDE from it.
template <class T>
__device__ __forceinline__ const T* opaque(const T* p) {
    asm("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

// sqrt.approx.ftz.f32 (one MUFU.SQRT; relative error ~2^-23, exactly 0 at 0)
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// t-th int16 offset (sign-extended) of a neighbour quad.
__device__ __forceinline__ int quad_offset(uint2 w, int t) {
    const uint32_t h = (t & 2) ? w.y : w.x;
    return (t & 1) ? ((int)h >> 16) : (int)(int16_t)(h & 0xffffu);
}

__device__ __forceinline__ void set_status(RolloutState* rs, int code, int particle) {
    if (atomicCAS(&rs->status, 0, code) == 0) {
        rs->bad_step = rs->step;
        rs->bad_particle = particle;
    }
}

// Enumerate the fluid candidates of a particle whose (rebuild-time) cell is c: the three cell
// rows cy-1..cy+1, each a contiguous slot range [start(cx-1), start(cx+2)) because cells are
// numbered row-major and slots are sorted by cell.
template <class F>
__device__ __forceinline__ void for_cell_candidates(const DevParams& P, const uint32_t* cs,
                                                    uint32_t c, F&& f) {
    int cy = (int)c / P.nx;
    int cx = (int)c - cy * P.nx;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
        int c0 = (cy + dy) * P.nx + cx - 1;
        uint32_t j0 = cs[c0], j1 = cs[c0 + 3];   // global or shared table
        for (uint32_t j = j0; j < j1; ++j) f(j);
    }
}

// Enumerate the fluid candidates of slot i (local index in its rollout): the neighbour list,
// or the rebuild-time cell block when the list overflowed.  f(j) gets local slot indices
// j != i.
template <class F>
__device__ __forceinline__ void for_fluid_candidates(const DevParams& P, const DevPtrs& D,
                                                     int b, int i, F&& f) {
    const size_t o = (size_t)b * P.N;
    const int n = D.ncnt[o + i];
    if (n != NL_OVERFLOW) {
        const uint2* nq = D.nbr + (size_t)b * KQ * P.N + i;
        for (int k = 0; k < n; ++k) f((uint32_t)(i + quad_offset(__ldg(nq + (k >> 2) * P.N), k & 3)));
    } else {
        for_cell_candidates(P, D.cstart + (size_t)b * (P.ncell + 1), D.skey[o + i],
                            [&](uint32_t j) {
                                if (j != (uint32_t)i) f(j);
                            });
    }
}

// Enumerate the candidate ghosts of a particle (ghost-ring lookup).  The ghosts sit uniformly
// on the wall circle, so those within 2h of x lie in an angular window around
// the particle's polar angle; the window half-width K (ghost_K for support 2h, ghost_K1 for
// support h) is derived on the host from |x - g|^2 >= 4 d R sin^2(dphi / 2) with
// d >= sqrt(wall_r2).  Exact predicates follow.
template <class F>
__device__ __forceinline__ void for_ghost_candidates(const DevParams& P, const Geom& gm,
                                                     float2 x, int K, float wall_r2, F&& f) {
    float rx = x.x - gm.rx, ry = x.y - gm.ry;
    if (rx * rx + ry * ry <= wall_r2) return;
    if (P.ghost_full) {
        for (int g = 0; g < P.G; ++g) f(g);
        return;
    }
    float phi = atan2f(ry, rx) - gm.th;
    int j0 = __float2int_rn(phi * P.ghost_scale) % P.G;
    if (j0 < 0) j0 += P.G;
    int g = j0 - K;
    if (g < 0) g += P.G;
    for (int t = 0; t < 2 * K + 1; ++t) {
        f(g);
        if (++g == P.G) g = 0;
    }
}

}  // namespace sph
