// sph_api.cu -- host side of libsphb200.so: the C ABI of include/sph.h.
// Validation, workspace carve-up, launch sequencing, CUDA-graph capture of a slow tick,
// canonical-order import/export and the parity/debug entry points.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/sph.h"
#include "sph_kernels.cuh"
#include "sph_resident.cuh"
#include "sph_jac.cuh"
#include "sph_calib.cuh"

using namespace sph;

struct sph_ctx {
    DevParams P;
    DevPtrs D;
    sph_fluid_params fp;   // float64 parameters as given (linearization works in float64)
    sph_body_params bp;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    float ghost_angle0 = 0.f;
    std::string err;
    // graph of one slow tick's substeps (n_sub substeps, damping 1, body free)
    cudaGraphExec_t tick_graph = nullptr;
    // staging for host-pointer calls (ctx-owned)
    void* stage = nullptr;
    size_t stage_bytes = 0;
    int* dbg_buf = nullptr;
    int n_sub = 1;
    int body_threads = BODY_T;   // k_body block size (from N only: reduction order fixed)
    // small-rollout rebuild path: k_rebuild_small on a forked branch (side stream + events)
    bool small = false;
    size_t small_smem = 0;
    int small_grid = 0;
    cudaStream_t side = nullptr;
    cudaStream_t side2 = nullptr;   // capture of the IF node's body (multi-kernel path)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool fork = true;   // small path: rebuild branch concurrent with density/forces
    bool pdl = true;    // programmatic dependent launch on the substep chain
    bool m2side = true; // small path: forces of the rebuilt rollouts at the end of the rebuild
                        // branch (overlapping the others' forces)
    float damping_cur = 1.0f;
    // execution path of a tick (sph_time_params.exec_path): 1 per-substep kernels, 2 cooperative
    // tick, 3 rollout-resident clusters
    int exec = 1;
    ResParams res{};     // resident path: cluster shape and shared-memory carve-up
    int res_nt = 0;      // resident path: threads per CTA
    cudaEvent_t res_ev[2] = {nullptr, nullptr};
    // small batches: the substep loop of a tick as one cooperative launch (k_coop)
    bool coop = false;
    int coop_grid = 0;
    // live kernel timing inside the tick graph (sph_set_live_timing): event-record nodes around
    // the density / force launches of every live_every-th substep, read after each tick
    int live_every = 0;
    std::vector<cudaEvent_t> live_ev;   // [sampled substep][LIVE_SLOTS]
    double live_ms[SPH_NUM_LIVE] = {0, 0, 0, 0};
    int64_t live_n = 0;
    // linearization scratch (sph_jacobian), kept between calls
    void* jac_buf = nullptr;
    size_t jac_bytes = 0;
    // dense eigensolver (sph_eigenvalues: cuSOLVER Xgeev, library call)
    cusolverDnHandle_t solver = nullptr;
    cusolverDnParams_t solver_params = nullptr;
    void* eig_dbuf = nullptr;
    size_t eig_dbytes = 0;
    std::vector<char> eig_hbuf;
    double* g1_buf = nullptr;   // sph_gamma1_estimate: (numerator, denominator) sums
};

// event slots of one sampled substep
enum { LV_SUB0 = 0, LV_DEN0, LV_DEN1, LV_F1_0, LV_F1_1, LV_F2_0, LV_F2_1, LV_SUB1, LIVE_SLOTS };

static std::string g_init_err;
static const int kSmallMinBatch = 512;   // auto policy: per-rollout-CTA rebuild from this B on

#define CK(expr)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (expr);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            ctx->err = std::string(#expr) + ": " + cudaGetErrorString(e_);             \
            return SPH_ECUDA;                                                          \
        }                                                                              \
    } while (0)

static sph_status fail(sph_ctx* ctx, sph_status s, const std::string& m) {
    if (ctx) ctx->err = m;
    else g_init_err = m;
    return s;
}

// Kernel launch, optionally with programmatic dependent launch (PDL): the kernel may start
// launching while its in-stream predecessor still runs; it waits (griddepcontrol.wait) before
// touching the predecessor's results.
template <typename... KArgs, typename... Args>
static void launch_k(bool pdl, void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                     Args... args) {
    if (!pdl) {
        kern<<<g, b, smem, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---------------------------------------------------------------------------------------
// Parameters and layout
// ---------------------------------------------------------------------------------------
static bool make_params(const sph_fluid_params* fp, const sph_body_params* bp,
                        const sph_time_params* tp, int N, int G, int B, DevParams* P,
                        std::string* why) {
    if (!fp || !bp || !tp) return *why = "null parameter struct", false;
    if (N < 0 || G < 0 || B < 1) return *why = "n_fluid, n_ghost must be >= 0, n_rollouts >= 1", false;
    if (!(fp->h > 0) || !(fp->rho0 > 0) || !(fp->mass > 0) || !(fp->k >= 0) ||
        !(fp->gamma1 > 0 && fp->gamma1 <= 1) || !(fp->eps > 0) || !(fp->alpha >= 0) ||
        !(fp->beta >= 0) || !(fp->w_cb_const > 0) || !std::isfinite(fp->gravity[0]) ||
        !std::isfinite(fp->gravity[1]))
        return *why = "invalid fluid parameters (h, rho0, mass > 0, k >= 0, gamma1 in (0,1], eps > 0, alpha, beta >= 0)", false;
    if (!(bp->m > 0) || !(bp->J > 0) || !(bp->tank_radius > 0))
        return *why = "invalid body parameters (m, J, tank_radius > 0)", false;
    if (!(tp->dt > 0) || tp->substeps_per_sample < 1 || tp->rebin_every < 0 || tp->rebin_every > 1 ||
        !(tp->skin >= 0))
        return *why = "invalid time parameters (dt > 0, substeps_per_sample >= 1, rebin_every in {0,1}, skin >= 0)", false;
    if (tp->rebuild_path < 0 || tp->rebuild_path > 2)
        return *why = "rebuild_path must be 0 (auto), 1 (per-rollout CTA) or 2 (multi-kernel)", false;
    if (tp->exec_path < 0 || tp->exec_path > 3)
        return *why = "exec_path must be 0 (auto), 1 (per-substep kernels), 2 (cooperative tick) or 3 (resident clusters)", false;
    if (tp->rebin_every == 0 && !(tp->skin > 0))
        return *why = "adaptive rebinning (rebin_every = 0) needs skin > 0", false;
    const double h = fp->h, R = bp->tank_radius;
    std::memset(P, 0, sizeof(*P));
    P->N = N;
    P->G = G;
    P->B = B;
    if (!(tp->skin_max >= 0.0) || (tp->skin_max > 0.0 && tp->skin_max < tp->skin))
        return *why = "skin_max must be 0 (fixed skin) or >= skin", false;
    if (tp->skin_mode < 0 || tp->skin_mode > 1) return *why = "skin_mode must be 0 or 1", false;
    const bool perpart = !tp->rebin_every && tp->skin_mode == 1 && tp->skin_max > tp->skin;
    const double skin_cell = tp->rebin_every ? 0.0 : std::max(tp->skin, tp->skin_max);
    const double Cd = 2.0 * h + skin_cell;
    P->C = (float)Cd;
    P->inv_C = 1.0f / P->C;
    const int half_cells = (int)std::ceil(R / (double)P->C) + 2;
    P->nx = 2 * half_cells;
    if ((double)P->nx * P->nx > 2.0e9 / std::max(B, 1))
        return *why = "cell grid too large", false;
    P->ncell = P->nx * P->nx;
    P->half = (float)half_cells * P->C;
    P->ntile = std::max(1, (N + TILE - 1) / TILE);
    P->npart = P->ntile * (TILE / 32);
    P->bsplit = P->npart > 8192 ? (P->npart + 511) / 512 : 1;
    P->own_lo = 0;
    P->own_n = N;
    P->nscan = (P->ncell + 1 + SCAN_TILE - 1) / SCAN_TILE;
    if ((P->nscan + SCAN_T - 1) / SCAN_T > SCAN_V) return *why = "cell grid too large for the scan", false;
    P->h = (float)h;
    P->inv_h = (float)(1.0 / h);
    const float H = (float)(2.0 * h);
    P->H2 = H * H;                        // float32 (2h)^2 (reading A19)
    P->h2 = P->h * P->h;
    P->mass = (float)fp->mass;
    P->m2 = (float)(fp->mass * fp->mass);
    P->rho0 = (float)fp->rho0;
    P->k = (float)fp->k;
    P->clampP = fp->clamp_negative_pressure != 0.0 ? 1 : 0;
    P->gamma1 = (float)fp->gamma1;
    P->alpha2h = (float)(2.0 * fp->alpha * h);
    P->beta = (float)fp->beta;
    P->eps_h2 = (float)(fp->eps * h * h);
    P->wcb = (float)(fp->w_cb_const / (h * h));
    P->dwcb = (float)(fp->w_cb_const / (h * h * h));
    P->mdwcb3 = (float)(fp->mass * 3.0 * fp->w_cb_const / (h * h * h));
    P->inv_mass = (float)(1.0 / fp->mass);
    P->dws3 = (float)(-30.0 / (M_PI * std::pow(h, 5)));
    P->gsign2m2 = (float)(fp->ghost_pressure_sign * 2.0 * fp->mass * fp->mass);
    P->gx = (float)fp->gravity[0];
    P->gy = (float)fp->gravity[1];
    P->dt = (float)tp->dt;
    P->dtd = tp->dt;
    P->m_body = bp->m;
    P->J_body = bp->J;
    P->rebin_every = tp->rebin_every;
    // list radius fl(2h + skin)^2 and rebuild threshold 0.49 skin per rollout (skin_set, B4 / B5)
    P->h2d = 2.0 * h;
    P->skin0 = tp->rebin_every ? 0.0f : (float)tp->skin;
    P->skin_max = tp->rebin_every ? 0.0f : (float)tp->skin_max;
    P->perpart = perpart ? 1 : 0;                    // per-particle half-skins (B6)
    P->Hf = H;
    P->hs_min = (float)(0.5 * tp->skin);
    P->hs_max = (float)(0.5 * tp->skin_max);
    P->hs_k = (float)(HS_TARGET * tp->dt);
    P->NA = (N + 1) & ~1;
    {   // CTA sizes of the plain density / force / list kernels.  Small CTAs win (C3 sweeps,
        // DESIGN.md section 7): a CTA's slot frees only when its slowest warp ends, and list
        // lengths / wall work differ from warp to warp.
        P->td = N >= 65536 ? 512 : 128;   // large tanks (C4: 10.70 -> 10.83 G/s, r02.46)
        // 128-slot force CTAs (r02.47 / r02.52: C4 10.81 -> 10.95 G/s, C3 94.97 -> 93.39 ms per
        // tick on the round-2 graph; 64 won on the round-1 graph, 256 loses on both)
        P->tf = 128;
        P->tn = 128;
        // k_force walks the rollouts last to first (L2 reuse after k_density; C3 A/B: force
        // 327.3 -> 326.5 us live, same bits)
        P->snake = 1;
        // L2 prefetch 1.5 waves ahead (a wave = 148 SMs x resident CTAs per SM at 48 (force) /
        // 64 (density) warps per SM; sweep: 0.5 16.7, 1 17.1, 1.5 17.2, 2 17.2, 4 16.8 G/s)
        P->pf_f = (int)(1.5 * 148 * (48 / (P->tf / 32)));
        P->pf_d = (int)(1.5 * 148 * (64 / (P->td / 32)));
    }
    // ghost-ring window (see for_ghost_candidates): only particles farther than d_min from the
    // centre can have a ghost within 2h; their ghosts lie within +-dphi of their polar angle.
    // |x - g| < s with |x| = d, |g| = R  =>  d > R - s  and  sin(dphi/2) < s / (2 sqrt(d R)).
    P->ghost_scale = (float)(G / (2.0 * M_PI));
    P->ghost_full = 1;
    P->wall_r2 = -1.0f;
    P->wall1_r2 = -1.0f;
    auto window = [&](double support, int* K, float* wall) {
        const double d_min = R - support - 1e-3 * h;
        if (!(G > 0 && d_min > 0)) return false;
        const double arg = support / (2.0 * std::sqrt(d_min * R));
        if (!(arg < 1.0)) return false;
        const double dphi = 2.0 * std::asin(arg);
        // ghost j lies at index distance |j - c| < dphi G / 2pi from the particle's continuous
        // index c = (atan2 - th) G / 2pi; the walk centres on j0 = round(c) (|c - j0| <= 1/2);
        // 0.05 index units (3e-4 rad at C2) cover the float error of atan2f / th / the body
        // position (~1e-6 rad).  (The ghost-set tests compare against brute force.)
        *K = (int)std::ceil(dphi * G / (2.0 * M_PI) + 0.5 + 0.05);
        *wall = std::nextafter((float)(d_min * d_min), 0.0f);
        return 2 * *K + 1 < G;
    };
    if (window(2.0 * h, &P->ghost_K, &P->wall_r2) && window(h, &P->ghost_K1, &P->wall1_r2))
        P->ghost_full = 0;
    return true;
}

// Workspace carve-up: one pass computes the offsets (base == nullptr) or binds the pointers.
static size_t carve(const DevParams& P, char* base, DevPtrs* D) {
    size_t o = 0;
    const size_t BN = (size_t)P.B * P.N, BG = (size_t)P.B * P.G;
    auto put = [&](auto*& ptr, size_t bytes) {
        using T = std::remove_reference_t<decltype(*ptr)>;
        ptr = base ? reinterpret_cast<T*>(base + o) : nullptr;
        o += (bytes + 255) & ~(size_t)255;
    };
    DevPtrs d{};
    put(d.pv[0], BN * 16);
    put(d.pv[1], BN * 16);
    put(d.id[0], BN * 4);
    put(d.id[1], BN * 4);
    put(d.aux, (size_t)P.B * P.NA * 8);   // rows of NA (even) elements: 16-B aligned
    put(d.skey, BN * 4);
    put(d.xb, BN * 8);
    put(d.hs, P.perpart ? BN * 4 : 4);
    put(d.nbr, BN * KQ * 8);
    put(d.ncnt, BN);
    put(d.key, BN * 4);
    put(d.rank, BN * 4);
    put(d.perm, BN * 4);
    put(d.counts, (size_t)P.B * P.ncell * 4);
    put(d.cstart, (size_t)P.B * (P.ncell + 1) * 4);
    put(d.tsum, (size_t)P.B * P.nscan * 4);
    put(d.gst, BG * 16);
    put(d.glo, BG * 8);
    put(d.garm, BG * 8);
    put(d.ghost_b, (size_t)std::max(P.G, 1) * 16);
    put(d.body, (size_t)P.B * 48);
    put(d.body_cs, (size_t)P.B * 16);
    put(d.u_cur, (size_t)P.B * 12);
    put(d.part, (size_t)P.B * P.npart * 32);
    put(d.part2, (size_t)P.B * P.bsplit * 32);
    put(d.rs, (size_t)P.B * sizeof(RolloutState));
    put(d.geom, (size_t)P.B * sizeof(Geom));
    put(d.xfer, (size_t)std::max(P.N, 1) * 16);
    put(d.xrho, (size_t)std::max(P.N, 1) * 4);
    put(d.rlist, (size_t)P.B * 4);
    put(d.rcount, 4);
    d.dbg_cnt = nullptr;
    d.dbg_idx = nullptr;
    if (D) *D = d;
    return o;
}

// ---------------------------------------------------------------------------------------
// Launch sequencing
// ---------------------------------------------------------------------------------------
static void launch_density(sph_ctx* ctx, cudaStream_t s, int skip_rebuilding, bool pdl = false) {
    pdl = pdl && ctx->pdl;
    const DevParams& P = ctx->P;
    switch (P.td) {
            case 1024: launch_k(pdl, k_density<1024>, dim3(std::max(1, (P.own_n + 1023) / 1024), P.B), dim3(1024), 0, s, P, ctx->D, skip_rebuilding); break;
            case 512: launch_k(pdl, k_density<512>, dim3(std::max(1, (P.own_n + 511) / 512), P.B), dim3(512), 0, s, P, ctx->D, skip_rebuilding); break;
            case 128: launch_k(pdl, k_density<128>, dim3(std::max(1, (P.own_n + 127) / 128), P.B), dim3(128), 0, s, P, ctx->D, skip_rebuilding); break;
            case 64: launch_k(pdl, k_density<64>, dim3(std::max(1, (P.own_n + 63) / 64), P.B), dim3(64), 0, s, P, ctx->D, skip_rebuilding); break;
            default: launch_k(pdl, k_density<256>, dim3(std::max(1, (P.own_n + 255) / 256), P.B), dim3(256), 0, s, P, ctx->D, skip_rebuilding); break;
        }
}

// mode: 0 all rollouts, 1 non-rebuilding rollouts, 2 rebuilt rollouts (work list)
static void launch_force(sph_ctx* ctx, cudaStream_t s, float damping, int mode = 0, bool pdl = false) {
    pdl = pdl && ctx->pdl;
    const DevParams& P = ctx->P;
    const int gy = mode == 2 ? std::min(P.B, 64) : P.B;
    // P.tf-slot CTAs (128, DESIGN.md r02.52); the per-particle-skin epilogue (B6) only in its own instance
#define SPH_FRC(TF)                                                                                \
    {                                                                                              \
        const dim3 g(std::max(1, (P.own_n + TF - 1) / TF), gy);                                    \
        if (P.perpart) launch_k(pdl, k_force<TF, true>, g, dim3(TF), 0, s, P, ctx->D, damping, mode);   \
        else launch_k(pdl, k_force<TF, false>, g, dim3(TF), 0, s, P, ctx->D, damping, mode);           \
    }
    switch (P.tf) {
        case 256: SPH_FRC(256); break;
        case 128: SPH_FRC(128); break;
        default: SPH_FRC(64); break;
    }
#undef SPH_FRC
}

static void launch_body(sph_ctx* ctx, cudaStream_t s, int pin, float ghost_angle0, bool pdl = false) {
    pdl = pdl && ctx->pdl;
    if (ctx->P.bsplit > 1) {   // (with PDL measured slower on C4: 207.5 vs 204.6 ms / tick)
        k_body_reduce<<<dim3(ctx->P.bsplit, ctx->P.B), BRED_T, 0, s>>>(ctx->P, ctx->D);
        pdl = false;
    }
    // large tanks in small batches (C4): the ghost update spread over k_ghosts' CTAs
    const int split = (ctx->P.B < 148 && ctx->P.G >= 4 * ctx->body_threads) ? 1 : 0;
    launch_k(pdl, k_body, dim3(ctx->P.B), dim3(ctx->body_threads), (size_t)ctx->body_threads * sizeof(double4),
             s, ctx->P, ctx->D, pin, ghost_angle0, split ^ 1);
    if (split)
        launch_k(pdl, k_ghosts, dim3((ctx->P.G + GH_T - 1) / GH_T, ctx->P.B), dim3(GH_T), 0, s, ctx->P, ctx->D);
}

// Grid-wide counting sort by cell of every rollout with need_rebin (7 kernels); with_nlist adds
// the grid-wide list build (debug path; the step uses k_nlist_density instead).
static void launch_rebin(sph_ctx* ctx, cudaStream_t s = nullptr, bool with_nlist = false) {
    const DevParams& P = ctx->P;
    if (!s) s = ctx->stream;
    dim3 gp(P.ntile, P.B), gs(P.nscan, P.B), gc((P.ncell + TILE - 1) / TILE, P.B);
    k_hash<<<gp, TILE, 0, s>>>(P, ctx->D);
    k_scan_reduce<<<gs, SCAN_T, 0, s>>>(P, ctx->D);
    k_scan_tiles<<<P.B, SCAN_T, 0, s>>>(P, ctx->D);
    k_scan_down<<<gs, SCAN_T, 0, s>>>(P, ctx->D);
    k_scatter<<<gp, TILE, 0, s>>>(P, ctx->D);
    k_cellsort<<<gc, TILE, 0, s>>>(P, ctx->D);
    k_gather<<<gp, TILE, 0, s>>>(P, ctx->D);
    if (with_nlist) k_nlist<<<gp, TILE, 0, s>>>(P, ctx->D);
}

// lists + densities of the rebuilt rollouts (work list), spread over the whole GPU: grid.y
// work-list slots (CTAs beyond the count return at once).  128 slots: the horizon's steady
// state (~260 rebuilding rollouts per substep) 13.37 -> 13.61 G/s against 64, the calm window
// unchanged (256: 13.68 / slightly slower window; 16 / 32: slower in both, DESIGN.md r02.30)
static void launch_nlist_density(sph_ctx* ctx, cudaStream_t s, bool pdl = false) {
    const DevParams& P = ctx->P;
    const int gy = std::min(P.B, 128);
    pdl = pdl && ctx->pdl;
    // the per-particle half-skin list radius (B6) only in its own instances
#define SPH_NLD(TN)                                                                                 \
    (P.perpart ? launch_k(pdl, k_nlist_density<TN, true>, dim3(std::max(1, (P.own_n + TN - 1) / TN), gy), \
                          dim3(TN), 0, s, P, ctx->D)                                                \
               : launch_k(pdl, k_nlist_density<TN, false>, dim3(std::max(1, (P.own_n + TN - 1) / TN), gy), \
                          dim3(TN), 0, s, P, ctx->D))
    switch (P.tn) {
        case 256: SPH_NLD(256); break;
        case 64: SPH_NLD(64); break;
        default: SPH_NLD(128); break;
    }
#undef SPH_NLD
}

// Rebuild (only rollouts that need it) + densities.  Small path: the plan kernel builds the
// work list, then k_rebuild_small (one CTA per rebuilding rollout, side stream) runs
// concurrently with k_density for every other rollout (fork/join via events; captured into
// the tick graph as two parallel branches).
// Multi-kernel path inside a graph capture: the plan kernel sets a conditional handle and the
// eight grid-wide rebuild kernels sit in the body of an IF node (skipped when no rollout of
// the batch needs a rebuild this substep).
static cudaError_t add_conditional_rebin(sph_ctx* ctx, cudaStream_t s) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
    if (e != cudaSuccess) return e;
    cudaGraphConditionalHandle h;
    if ((e = cudaGraphConditionalHandleCreate(&h, g, 0, 0)) != cudaSuccess) return e;
    k_rebuild_plan<<<1, RB_T, 0, s>>>(ctx->P, ctx->D, h, 1);
    if ((e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd)) != cudaSuccess) return e;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, deps, nd, &cp)) != cudaSuccess) return e;
    if ((e = cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
        return e;
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(ctx->side2, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return e;
    launch_rebin(ctx, ctx->side2);
    // lists + densities of the rebuilt rollouts inside the IF body too: substeps without a
    // rebuild then launch no list kernel at all (C4: one launch of ~8,000 empty CTAs less per
    // substep); they only touch rebuilt rollouts, k_density the others (disjoint), so running
    // them before k_density changes nothing
    launch_nlist_density(ctx, ctx->side2);
    return cudaStreamEndCapture(ctx->side2, &body);
}

// Rebuild (only rollouts that need it) + densities.  Small path: the plan kernel builds the
// work list, then k_rebuild_small (one CTA per rebuilding rollout, side stream) runs
// concurrently with k_density for every other rollout (fork/join via events; captured into
// the tick graph as two parallel branches).  Multi-kernel path: grid-wide rebuild kernels,
// under an IF node when captured.
// Timing mark of a live-timed substep (ev == nullptr: not sampled).  Only used while capturing
// the tick graph: an external event record becomes an event-record node of the graph.
static void live_mark(cudaEvent_t* ev, int slot, cudaStream_t s) {
    if (ev) cudaEventRecordWithFlags(ev[slot], s, cudaEventRecordExternal);
}

// first: the substep's first kernel has an in-stream kernel predecessor (PDL allowed); timing
// nodes (ev) between kernels disable PDL for the kernels after them.
static cudaError_t launch_rebuild_and_density(sph_ctx* ctx, bool capturing, cudaEvent_t* ev,
                                              bool first_pdl) {
    const DevParams& P = ctx->P;
    cudaStream_t s = ctx->stream;
    dim3 gp(P.ntile, P.B);
    const bool np = ev == nullptr;   // no timing nodes in this substep
    if (ctx->small && !ctx->fork) {   // serial: sort + lists/densities of the rebuilt rollouts first
        k_rebuild_plan<<<1, RB_T, 0, s>>>(P, ctx->D, 0, 0);
        k_rebuild_small<<<ctx->small_grid, RBS_T, ctx->small_smem, s>>>(P, ctx->D);
        launch_nlist_density(ctx, s);
        live_mark(ev, LV_DEN0, s);
        launch_density(ctx, s, 1);
        live_mark(ev, LV_DEN1, s);
        return cudaSuccess;
    }
    if (ctx->small) {   // (forces are launched by launch_substep, see there)
        // the plan kernel heads the rebuild branch: k_density / mode-1 forces read need_rebin
        // themselves, only the branch needs the work list
        cudaEventRecord(ctx->ev_fork, s);
        cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
        k_rebuild_plan<<<1, RB_T, 0, ctx->side>>>(P, ctx->D, (cudaGraphConditionalHandle)0, 0);
        k_rebuild_small<<<ctx->small_grid, RBS_T, ctx->small_smem, ctx->side>>>(P, ctx->D);
        launch_nlist_density(ctx, ctx->side, true);
        if (ctx->m2side) {   // (timing nodes on the side stream: the force time is the sum
                             // of both launches' durations)
            live_mark(ev, LV_F2_0, ctx->side);
            launch_force(ctx, ctx->side, ctx->damping_cur, 2, np);
            live_mark(ev, LV_F2_1, ctx->side);
        }
        cudaEventRecord(ctx->ev_join, ctx->side);
        live_mark(ev, LV_DEN0, s);
        launch_density(ctx, s, 1, np);
        live_mark(ev, LV_DEN1, s);
        return cudaSuccess;
    } else {
        if (capturing) {
            // plan + IF node on a forked branch, concurrent with the densities of the rollouts
            // that do not rebuild (disjoint rollouts, as on the small path): the IF node's own
            // scheduling cost (~7 us per substep, tools/micro/ifnode.cu) hides under k_density
            cudaEventRecord(ctx->ev_fork, s);
            cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
            cudaError_t e = add_conditional_rebin(ctx, ctx->side);
            if (e != cudaSuccess) return e;
            cudaEventRecord(ctx->ev_join, ctx->side);
            live_mark(ev, LV_DEN0, s);
            launch_density(ctx, s, 1, np);
            live_mark(ev, LV_DEN1, s);
            cudaStreamWaitEvent(s, ctx->ev_join, 0);
            return cudaSuccess;
        } else {
            k_rebuild_plan<<<1, RB_T, 0, s>>>(P, ctx->D, 0, 0);
            launch_rebin(ctx);
        }
        live_mark(ev, LV_DEN0, s);
        launch_density(ctx, s, 1, false);   // (follows the IF node / the rebuild kernels)
        live_mark(ev, LV_DEN1, s);
        if (capturing) return cudaSuccess;   // (lists inside the IF body, add_conditional_rebin)
    }
    launch_nlist_density(ctx, s, np);
    return cudaSuccess;
}

// k = substep index inside the captured tick (live timing samples every live_every-th one)
static cudaError_t launch_substep(sph_ctx* ctx, float damping, int pin, bool capturing = false,
                                  int k = -1) {
    const DevParams& P = ctx->P;
    cudaStream_t s = ctx->stream;
    dim3 gp(P.ntile, P.B);
    cudaEvent_t* ev = nullptr;
    if (capturing && ctx->live_every > 0 && k >= 0 && k % ctx->live_every == 0)
        ev = ctx->live_ev.data() + (size_t)(k / ctx->live_every) * LIVE_SLOTS;
    live_mark(ev, LV_SUB0, s);
    const bool np = ev == nullptr;
    ctx->damping_cur = damping;   // (the rebuild branch launches the rebuilt rollouts' forces)
    // PDL on the first kernel only when an in-stream kernel precedes it (not the first substep
    // of a captured graph)
    cudaError_t e = launch_rebuild_and_density(ctx, capturing, ev, !(capturing && k == 0));
    if (ctx->small && ctx->fork) {
        // The rebuild branch (sort -> lists + densities of the rebuilt rollouts) runs on the side
        // stream concurrently with density AND forces of every other rollout; only the forces
        // of the rebuilt rollouts wait for it.
        live_mark(ev, LV_F1_0, s);
        launch_force(ctx, s, damping, 1, np);
        live_mark(ev, LV_F1_1, s);
        cudaStreamWaitEvent(s, ctx->ev_join, 0);
        if (!ctx->m2side) {
            live_mark(ev, LV_F2_0, s);
            launch_force(ctx, s, damping, 2, false);
            live_mark(ev, LV_F2_1, s);
        }
    } else {
        live_mark(ev, LV_F1_0, s);
        launch_force(ctx, s, damping, 0, np);
        live_mark(ev, LV_F1_1, s);
    }
    launch_body(ctx, s, pin, ctx->ghost_angle0, np);
    live_mark(ev, LV_SUB1, s);
    return e;
}

// n substeps of the small-batch path in one cooperative launch
static cudaError_t launch_coop(sph_ctx* ctx, int n, float damping, int pin) {
    DevParams P = ctx->P;
    DevPtrs D = ctx->D;
    float ga = ctx->ghost_angle0;
    int nt = ctx->body_threads;
    void* args[] = {&P, &D, &n, &damping, &pin, &ga, &nt};
    return cudaLaunchCooperativeKernel((void*)k_coop, dim3(ctx->coop_grid), dim3(COOP_T), args, 0,
                                       ctx->stream);
}

static int live_samples(const sph_ctx* ctx) {
    return ctx->live_every > 0 ? (ctx->n_sub + ctx->live_every - 1) / ctx->live_every : 0;
}

// kernels per substep: small path 5 (plan, rebuild_small, density, force, body); multi-kernel
// path 4 + 8 rebuild kernels (the 8 run only in substeps where some rollout rebuilds).
static int launches_per_substep(const sph_ctx* ctx) {
    return (ctx->small ? (ctx->fork ? 7 : 6) : 12) + (ctx->P.bsplit > 1 ? 1 : 0) +
           ((ctx->P.B < 148 && ctx->P.G >= 4 * ctx->body_threads) ? 1 : 0);
}

static sph_status check_launch(sph_ctx* ctx) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, SPH_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    return SPH_OK;
}

static sph_status ensure_stage(sph_ctx* ctx, size_t bytes) {
    if (ctx->stage_bytes >= bytes) return SPH_OK;
    if (ctx->stage) cudaFree(ctx->stage);
    ctx->stage = nullptr;
    ctx->stage_bytes = 0;
    CK(cudaMalloc(&ctx->stage, bytes));
    ctx->stage_bytes = bytes;
    return SPH_OK;
}

static sph_status all_failed(sph_ctx* ctx) {
    std::vector<RolloutState> rs(ctx->P.B);
    CK(cudaMemcpyAsync(rs.data(), ctx->D.rs, sizeof(RolloutState) * ctx->P.B, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto& r : rs)
        if (!r.status) return SPH_OK;
    return fail(ctx, SPH_EBLOWUP, "every rollout has a non-zero numerical status");
}

// Raise (never lower) a kernel's dynamic shared-memory limit: the attribute is per function and
// process-wide, so a context must not shrink it under another context that needs more.
template <class K>
static cudaError_t raise_smem_limit(K kern, size_t bytes) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    if ((size_t)fa.maxDynamicSharedSizeBytes >= bytes) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ---------------------------------------------------------------------------------------
// Resident path (k_resident, sph_resident.cuh)
// ---------------------------------------------------------------------------------------
// Cluster shape and shared-memory carve-up for CS CTAs per rollout; false if it does not fit.
static bool res_layout(const DevParams& P, int CS, int smem_max, ResParams* out, int* nt_out) {
    if (P.N <= 0 || P.N >= 65536 || P.perpart) return false;   // (uniform / B5 skins only)
    ResParams R{};
    R.CS = CS;
    R.S = ((P.N + CS - 1) / CS + 31) / 32 * 32;
    if ((long long)(CS - 1) * R.S >= P.N) return false;          // every CTA owns slots
    const int units = R.S / 32;
    const int rounds = (units + RES_MAXT / 32 - 1) / (RES_MAXT / 32);
    if (rounds > RES_RU) return false;
    const int nt = 32 * ((units + rounds - 1) / rounds);
    if (R.S > RES_RU * nt) return false;
    int idb = 1;
    while ((1 << idb) < P.N) ++idb;
    R.IDB = idb;
    R.idmask = (1u << idb) - 1u;
    if (((unsigned long long)(P.ncell + 1) << idb) > 0xffffffffull) return false;
    // halo per side: one cell row + 3 cells at up to 8 particles per cell (rest lattice: 3.8 per
    // 2h + skin cell; the weakly compressible fluid stays below ~1.35 rho0)
    R.HCAP = std::min(((P.nx + 3) * 8 + 31) / 32 * 32, (CS - 1) * R.S);
    R.W = R.S + 2 * R.HCAP;
    if (R.W > 65535) return false;
    R.KR = 16;
    R.KQ = R.KR / 4;
    R.MCAP = 1024;
    R.NCT = P.ncell + 2;
    R.npart = (P.N + 31) / 32;
    int o = 0;
    auto put = [&](int* off, long long bytes) {
        *off = o;
        o += (int)((bytes + 15) & ~15ll);
    };
    put(&R.o_pv, 16ll * R.W);
    put(&R.o_rpv, 16ll * R.S);
    put(&R.o_gst, 16ll * std::max(P.G, 1));
    put(&R.o_glo, 16ll * std::max(P.G, 1));
    put(&R.o_ghb, 16ll * std::max(P.G, 1));
    put(&R.o_part, 32ll * R.npart);
    put(&R.o_aux, 8ll * R.W);
    put(&R.o_xb, 8ll * R.S);
    put(&R.o_nbr, 8ll * R.KQ * R.S);
    put(&R.o_key, 4ll * R.W);
    put(&R.o_rkey, 4ll * R.S);
    put(&R.o_nmk, 4ll * R.S);
    put(&R.o_obk, 4ll * R.S);
    put(&R.o_mkg, 4ll * R.MCAP);
    put(&R.o_mks, 4ll * R.MCAP);
    put(&R.o_wcs, 2ll * R.NCT);
    put(&R.o_obj, 2ll * R.S);
    put(&R.o_ncnt, R.S);
    put(&R.o_misc, sizeof(ResMisc));
    R.smem = o;
    if (R.smem > smem_max) return false;
    *out = R;
    *nt_out = nt;
    return true;
}

static cudaError_t launch_resident(sph_ctx* ctx, const TickArgs& T) {
    const DevParams& P = ctx->P;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.B * ctx->res.CS);
    cfg.blockDim = dim3(ctx->res_nt);
    cfg.dynamicSmemBytes = ctx->res.smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ctx->res.CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const bool timed = ctx->live_every > 0 && T.u_seq != nullptr;
    if (timed) cudaEventRecord(ctx->res_ev[0], ctx->stream);
#ifdef SPH_RES_TIMING
    // diagnostic build: per-CTA phase timestamps of this launch appended to $SPH_RES_TIMING_FILE
    // as [B * CS][n_sub][RES_NMARK] uint64 ns (header: CTAs, n_sub, RES_NMARK)
    TickArgs Tt = T;
    const size_t nclk = (size_t)P.B * ctx->res.CS * T.n_sub * RES_NMARK;
    cudaMalloc(&Tt.clk, nclk * 8);
    cudaMemsetAsync(Tt.clk, 0, nclk * 8, ctx->stream);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_resident, P, ctx->D, ctx->res, Tt);
    std::vector<unsigned long long> h(nclk);
    cudaMemcpyAsync(h.data(), Tt.clk, nclk * 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(Tt.clk);
    if (const char* fn = std::getenv("SPH_RES_TIMING_FILE")) {
        if (FILE* f = std::fopen(fn, "ab")) {
            const unsigned long long hdr[3] = {(unsigned long long)P.B * ctx->res.CS, (unsigned long long)T.n_sub,
                                               (unsigned long long)RES_NMARK};
            std::fwrite(hdr, 8, 3, f);
            std::fwrite(h.data(), 8, nclk, f);
            std::fclose(f);
        }
    }
#else
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_resident, P, ctx->D, ctx->res, T);
#endif
    if (timed) cudaEventRecord(ctx->res_ev[1], ctx->stream);
    return e;
}

static TickArgs hold_args(const sph_ctx* ctx, int n, float damping, int pin) {
    TickArgs T{};
    T.n_sub = n;
    T.damping = damping;
    T.pin = pin;
    T.ghost_angle0 = ctx->ghost_angle0;
    return T;
}

// Resident-path eligibility at init: the smallest cluster (1, 2, 4, 8, 16 CTAs per rollout)
// whose carve-up fits one CTA's shared memory and that the device can co-schedule.
static bool res_setup(sph_ctx* ctx) {
    int dev = 0, optin = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // latency-bound small batches (B x 16 CTAs fit the SMs): the widest cluster that fits, so a
    // substep's work spreads over the most SMs; otherwise the narrowest (least halo, fewest
    // barriers per particle)
    const bool wide = ctx->P.B * RES_MAXCS <= nsm;
    for (int k = 0; k < 5; ++k) {
        const int CS = wide ? (RES_MAXCS >> k) : (1 << k);
        ResParams R;
        int nt = 0;
        if (!res_layout(ctx->P, CS, optin, &R, &nt)) continue;
        if (raise_smem_limit(k_resident, R.smem) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (CS > 8 && cudaFuncSetAttribute(k_resident, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CS * std::max(ctx->P.B, 1));
        cfg.blockDim = dim3(nt);
        cfg.dynamicSmemBytes = R.smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_resident, &cfg) != cudaSuccess || ncl < 1) {
            cudaGetLastError();
            continue;
        }
        ctx->res = R;
        ctx->res_nt = nt;
        return true;
    }
    return false;
}

__global__ void k_force_rebin(RolloutState* rs, int b) { rs[b].need_rebin = 1; }

// ---------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------
extern "C" {

size_t sph_workspace_bytes(const sph_fluid_params* fp, const sph_body_params* bp,
                           const sph_time_params* tp, int n_fluid, int n_ghost, int n_rollouts) {
    DevParams P;
    std::string why;
    if (!make_params(fp, bp, tp, n_fluid, n_ghost, n_rollouts, &P, &why)) return 0;
    return carve(P, nullptr, nullptr);
}

sph_status sph_init_tank(const sph_fluid_params* fp, const sph_body_params* bp,
                         const sph_time_params* tp, int n_fluid, const float* fluid_pv,
                         int n_ghost, const double* ghost_body_xy, int n_rollouts,
                         void* cuda_stream, void* d_workspace, size_t workspace_bytes,
                         sph_ctx** out) {
    if (!out) return fail(nullptr, SPH_EINVAL, "out is NULL");
    *out = nullptr;
    DevParams P;
    std::string why;
    if (!make_params(fp, bp, tp, n_fluid, n_ghost, n_rollouts, &P, &why))
        return fail(nullptr, SPH_EINVAL, why);
    if ((n_fluid > 0 && !fluid_pv) || (n_ghost > 0 && !ghost_body_xy))
        return fail(nullptr, SPH_EINVAL, "fluid_pv / ghost_body_xy is NULL");
    const size_t total = carve(P, nullptr, nullptr);
    if (!d_workspace || workspace_bytes < total)
        return fail(nullptr, SPH_ENOMEM, "workspace too small: need " + std::to_string(total) + " bytes");
    if (((uintptr_t)d_workspace) & 255) return fail(nullptr, SPH_EINVAL, "workspace must be 256-byte aligned");
    for (int i = 0; i < 4 * n_fluid; ++i)
        if (!std::isfinite(fluid_pv[i])) return fail(nullptr, SPH_EINVAL, "non-finite fluid state");
    // the ghost-ring lookup needs ghosts uniformly spaced on the wall circle, angular order
    const double R = bp->tank_radius;
    double a0 = 0.0;
    if (n_ghost > 0) {
        a0 = std::atan2(ghost_body_xy[1], ghost_body_xy[0]);
        for (int g = 0; g < n_ghost; ++g) {
            const double a = a0 + 2.0 * M_PI * g / n_ghost;
            const double ex = R * std::cos(a) - ghost_body_xy[2 * g];
            const double ey = R * std::sin(a) - ghost_body_xy[2 * g + 1];
            if (std::sqrt(ex * ex + ey * ey) > 1e-6 * R)
                return fail(nullptr, SPH_EINVAL, "ghosts must lie uniformly spaced on the tank wall circle (radius tank_radius) in counter-clockwise order");
        }
    }
    sph_ctx* ctx = new sph_ctx();
    ctx->P = P;
    ctx->fp = *fp;
    ctx->bp = *bp;
    // PDL pays for latency-bound small batches (C1 / C2 single tank +4 %); at C3 it is
    // neutral to -1 %, so it is on below the per-rollout rebuild threshold only.
    ctx->pdl = P.B < kSmallMinBatch;
    ctx->n_sub = tp->substeps_per_sample;
    ctx->ghost_angle0 = (float)a0;
    carve(P, (char*)d_workspace, &ctx->D);
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete ctx;
            return fail(nullptr, SPH_ECUDA, "cudaStreamCreate failed");
        }
        ctx->own_stream = true;
    }
    cudaStream_t s = ctx->stream;
    auto bail = [&](const char* what, cudaError_t e) {
        g_init_err = std::string(what) + ": " + cudaGetErrorString(e);
        sph_destroy(ctx);
        return SPH_ECUDA;
    };
    cudaError_t e;
    // rebuild path: one CTA per rebuilding rollout when its cell table and sort scratch fit in
    // shared memory (rebuild_path 0 = auto, 1 = force per-rollout CTA, 2 = force multi-kernel)
    {
        const size_t smem = (size_t)((P.ncell + 1 + 3) & ~3) * 4 + (size_t)P.N * 14 + 16;
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const bool fits = P.N > 0 && P.N < 65536 && P.ncell < 65535 && smem <= 200 * 1024;
        // auto: the one-CTA rebuild of a rollout (~0.2 ms on one SM) hides under the densities
        // of the other rollouts only for large batches; small batches use the grid-wide
        // kernels (under a graph IF node).
        bool want = tp->rebuild_path == 1 || (tp->rebuild_path == 0 && fits && P.B >= kSmallMinBatch);
        if (want && !fits) {
            sph_destroy(ctx);
            return fail(nullptr, SPH_EINVAL, "rebuild_path = 1 but the rollout does not fit in shared memory");
        }
        if (want && raise_smem_limit(k_rebuild_small, smem) != cudaSuccess) {
            cudaGetLastError();
            want = false;
        }
        if (want) {
            ctx->small = true;
            ctx->small_smem = smem;
            ctx->small_grid = std::max(1, std::min(P.B, nsm));
        }
        if ((e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming)) != cudaSuccess)
            return bail("side stream", e);
        // k_body: enough threads to reduce the per-warp partials of big tanks (N only)
        while (ctx->body_threads < 1024 && ctx->body_threads * 4 < P.npart) ctx->body_threads *= 2;
        if (P.bsplit > 1) {   // k_body sums bsplit chunk sums: a power of two >= bsplit threads
            // (every slot holds at most one chunk sum, so the tree -- and the bits -- equal
            // the 1024-thread block's)
            int bt = 32;
            while (bt < P.bsplit && bt < 1024) bt *= 2;
            ctx->body_threads = bt;
        }
        {   // cooperative tick for latency-bound small batches (exec_path 2 forces it)
            bool want = tp->exec_path == 2 || (tp->exec_path == 0 && (size_t)P.B * P.N <= 65536 && !ctx->small);
            want = want && ctx->body_threads <= COOP_T && P.bsplit == 1;
            int coop_ok = 0, per_sm = 0;
            cudaDeviceGetAttribute(&coop_ok, cudaDevAttrCooperativeLaunch, dev);
            if (want && coop_ok &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coop, COOP_T, 0) == cudaSuccess &&
                per_sm > 0) {
                const int ncb = (P.ncell + TILE - 1) / TILE;
                const int need = std::max({P.ntile * P.B, ncb * P.B, P.nscan * P.B, P.B, 1});
                ctx->coop_grid = std::min(per_sm * nsm, need);
                ctx->coop = true;
            }
            cudaGetLastError();
        }
    }
    // resident clusters (exec_path 3, opt-in)
    ctx->exec = ctx->coop ? 2 : 1;
    // auto picks it for latency-bound small batches whose clusters all fit the GPU at once (B x
    // 16 CTAs <= SMs): C1 / C2 single tanks and P0 run 1.5-1.9x faster than the cooperative tick
    // (DESIGN.md 7b); for large batches the per-substep kernels win (one 19-warp CTA per SM and two
    // cluster barriers per substep cannot match their 40+ warps per SM)
    int nsm_ = 148, dev_ = 0;
    cudaGetDevice(&dev_);
    cudaDeviceGetAttribute(&nsm_, cudaDevAttrMultiProcessorCount, dev_);
    if (tp->exec_path == 3 || (tp->exec_path == 0 && (long long)P.B * RES_MAXCS <= nsm_)) {
        const bool ok = res_setup(ctx);
        if (!ok && tp->exec_path == 3) {
            sph_destroy(ctx);
            return fail(nullptr, SPH_EINVAL, "exec_path = 3 but the rollout does not fit a cluster's shared memory (n_fluid < 65536, one cell row of halo per CTA)");
        }
        if (ok) {
            ctx->exec = 3;
            ctx->coop = false;
            if ((e = cudaEventCreate(&ctx->res_ev[0])) != cudaSuccess ||
                (e = cudaEventCreate(&ctx->res_ev[1])) != cudaSuccess)
                return bail("resident events", e);
        }
    }
    if ((e = cudaMemsetAsync(d_workspace, 0, total, s)) != cudaSuccess) return bail("memset", e);
    std::vector<double2> gb(std::max(n_ghost, 1));
    for (int g = 0; g < n_ghost; ++g) gb[g] = make_double2(ghost_body_xy[2 * g], ghost_body_xy[2 * g + 1]);
    if (n_ghost > 0 && (e = cudaMemcpyAsync(ctx->D.ghost_b, gb.data(), sizeof(double2) * n_ghost, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return bail("ghost copy", e);
    if (n_fluid > 0) {
        if ((e = cudaMemcpyAsync(ctx->D.xfer, fluid_pv, sizeof(float4) * n_fluid, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return bail("state copy", e);
        k_import<<<dim3((n_fluid + 255) / 256, P.B), 256, 0, s>>>(P, ctx->D, 0, ctx->D.xfer);
    }
    k_reset_rollout<<<P.B, BODY_T, 0, s>>>(P, ctx->D, 0, ctx->ghost_angle0, 1);
    if ((e = cudaGetLastError()) != cudaSuccess) return bail("init kernels", e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail("init sync", e);
    *out = ctx;
    return SPH_OK;
}

sph_status sph_set_state(sph_ctx* ctx, int rollout, const float* fluid_pv, const double* body) {
    if (!ctx) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < -1 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    if (P.N > 0 && !fluid_pv) return fail(ctx, SPH_EINVAL, "fluid_pv is NULL");
    for (int i = 0; i < 4 * P.N; ++i)
        if (!std::isfinite(fluid_pv[i])) return fail(ctx, SPH_EINVAL, "non-finite fluid state");
    const int b0 = rollout < 0 ? 0 : rollout, nb = rollout < 0 ? P.B : 1;
    cudaStream_t s = ctx->stream;
    if (P.N > 0) {
        CK(cudaMemcpyAsync(ctx->D.xfer, fluid_pv, sizeof(float4) * P.N, cudaMemcpyHostToDevice, s));
        k_import<<<dim3(std::max(1, (P.N + 255) / 256), nb), 256, 0, s>>>(P, ctx->D, b0, ctx->D.xfer);
    }
    if (body) {
        for (int b = b0; b < b0 + nb; ++b)
            CK(cudaMemcpyAsync(ctx->D.body + (size_t)b * 6, body, 48, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemsetAsync(ctx->D.counts + (size_t)b0 * P.ncell, 0, sizeof(uint32_t) * P.ncell * nb, s));
    k_reset_rollout<<<nb, BODY_T, 0, s>>>(P, ctx->D, b0, ctx->ghost_angle0, 1);
    sph_status st = check_launch(ctx);
    if (st) return st;
    CK(cudaStreamSynchronize(s));
    return SPH_OK;
}

sph_status sph_set_body_state(sph_ctx* ctx, const double* body) {
    if (!ctx || !body) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    for (int i = 0; i < 6 * P.B; ++i)
        if (!std::isfinite(body[i])) return fail(ctx, SPH_EINVAL, "non-finite body state");
    CK(cudaMemcpyAsync(ctx->D.body, body, 48 * (size_t)P.B, cudaMemcpyHostToDevice, ctx->stream));
    // keep status / freeze / failure record, refresh ghosts and the float pose
    k_reset_rollout<<<P.B, BODY_T, 0, ctx->stream>>>(P, ctx->D, 0, ctx->ghost_angle0, 0);
    sph_status st = check_launch(ctx);
    if (st) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
}

sph_status sph_get_particles(sph_ctx* ctx, int rollout, float* fluid_pv, float* rho) {
    if (!ctx || !fluid_pv) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < 0 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    if (P.N == 0) return SPH_OK;
    cudaStream_t s = ctx->stream;
    k_export<<<(P.N + 255) / 256, 256, 0, s>>>(P, ctx->D, rollout, ctx->D.xfer, ctx->D.xrho);
    sph_status st = check_launch(ctx);
    if (st) return st;
    CK(cudaMemcpyAsync(fluid_pv, ctx->D.xfer, sizeof(float4) * P.N, cudaMemcpyDeviceToHost, s));
    if (rho) CK(cudaMemcpyAsync(rho, ctx->D.xrho, sizeof(float) * P.N, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return SPH_OK;
}

sph_status sph_gamma1_estimate(sph_ctx* ctx, int rollout, double rho_target, float* gamma1_i,
                               float* sums, double* gamma1_wall) {
    if (!ctx) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < 0 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    if (!(rho_target > 0.0)) return fail(ctx, SPH_EINVAL, "rho_target must be > 0");
    if (gamma1_wall) *gamma1_wall = std::nan("");
    if (P.N == 0) return SPH_OK;
    cudaStream_t s = ctx->stream;
    if (!ctx->g1_buf) CK(cudaMalloc(&ctx->g1_buf, 2 * sizeof(double)));
    // target density in units of m C / h^2, from the float64 parameters
    const double wcb = ctx->fp.w_cb_const / (ctx->fp.h * ctx->fp.h);
    const float rt = (float)(rho_target / (ctx->fp.mass * wcb));
    float2* parts = reinterpret_cast<float2*>(ctx->D.xfer);   // [N] staging (k_export's)
    k_gamma1_parts<<<(P.N + G1_T - 1) / G1_T, G1_T, 0, s>>>(P, ctx->D, rollout, rt, parts,
                                                           ctx->D.xrho);
    k_gamma1_wall<<<1, 1024, 0, s>>>(P.N, parts, rt, ctx->g1_buf);
    sph_status st = check_launch(ctx);
    if (st) return st;
    double nd[2];
    if (gamma1_i) CK(cudaMemcpyAsync(gamma1_i, ctx->D.xrho, sizeof(float) * P.N, cudaMemcpyDeviceToHost, s));
    if (sums) CK(cudaMemcpyAsync(sums, parts, sizeof(float2) * P.N, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(nd, ctx->g1_buf, sizeof(nd), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (gamma1_wall && nd[1] > 0.0) *gamma1_wall = nd[0] / nd[1];
    return SPH_OK;
}

sph_status sph_get_ghosts(sph_ctx* ctx, int rollout, float* ghost_pv) {
    if (!ctx || !ghost_pv) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < 0 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    if (P.G == 0) return SPH_OK;
    CK(cudaMemcpyAsync(ghost_pv, ctx->D.gst + (size_t)rollout * P.G, sizeof(float4) * P.G, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
}

sph_status sph_set_domain(sph_ctx* ctx, int slot_lo, int slot_hi) {
    if (!ctx) return SPH_EINVAL;
    DevParams& P = ctx->P;
    if (P.B != 1) return fail(ctx, SPH_EINVAL, "domain decomposition needs a single rollout");
    if (slot_lo < 0 || slot_hi <= slot_lo || slot_hi > P.N || slot_lo % SPH_DD_ALIGN != 0 ||
        (slot_hi != P.N && slot_hi % SPH_DD_ALIGN != 0))
        return fail(ctx, SPH_EINVAL, "slot range must be [lo, hi) within [0, N), lo and hi multiples of SPH_DD_ALIGN (hi may be N)");
    CK(cudaStreamSynchronize(ctx->stream));
    P.own_lo = slot_lo;
    P.own_n = slot_hi - slot_lo;
    // the per-substep kernel path with grid-wide rebuild kernels (no single-launch tick, no
    // per-rollout shared-memory sort, no ring kernels); graphs captured before are stale
    P.pf_d = P.pf_f = 0;
    ctx->coop = false;
    ctx->small = false;
    // the resident path persists its Verlet lists in shared memory only (rs->need_rebin may be 0
    // with no lists in global memory): the kernel path starts with a rebuild
    if (ctx->exec == 3) k_force_rebin<<<1, 1, 0, ctx->stream>>>(ctx->D.rs, 0);
    ctx->exec = 1;
    if (ctx->tick_graph) {
        cudaGraphExecDestroy(ctx->tick_graph);
        ctx->tick_graph = nullptr;
    }
    return SPH_OK;
}

sph_status sph_dd_phase(sph_ctx* ctx, int phase, const float* u, void* aux_io, void* state_io,
                        void* part_io) {
    if (!ctx || !aux_io || !state_io || !part_io || phase < 0 || phase > 2) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (P.B != 1) return fail(ctx, SPH_EINVAL, "domain decomposition needs a single rollout");
    if (P.N == 0) return SPH_OK;
    cudaStream_t s = ctx->stream;
    float2* aux = static_cast<float2*>(aux_io);
    float4* st = static_cast<float4*>(state_io);
    double4* part = static_cast<double4*>(part_io);
    const int lo = P.own_lo, n = P.own_n;
    const int q0 = lo / 32, q1 = std::min(P.npart, (lo + n + 31) / 32);
    if (phase == 0) {
        if (u) {
            for (int i = 0; i < 3; ++i)
                if (!std::isfinite(u[i])) return fail(ctx, SPH_EINVAL, "non-finite input u");
            CK(cudaMemcpyAsync(ctx->D.u_cur, u, sizeof(float) * 3, cudaMemcpyHostToDevice, s));
        }
        ctx->damping_cur = 1.0f;
        launch_rebuild_and_density(ctx, false, nullptr, false);
        CK(cudaMemcpyAsync(aux + lo, ctx->D.aux + lo, sizeof(float2) * n, cudaMemcpyDeviceToDevice, s));
    } else if (phase == 1) {
        CK(cudaMemcpyAsync(ctx->D.aux, aux, sizeof(float2) * P.N, cudaMemcpyDeviceToDevice, s));
        launch_force(ctx, s, 1.0f, 0, false);
        k_dd_export<<<(n + 255) / 256, 256, 0, s>>>(P, ctx->D, st);
        CK(cudaMemcpyAsync(part + q0, ctx->D.part + q0, sizeof(double4) * (q1 - q0), cudaMemcpyDeviceToDevice, s));
    } else {
        k_dd_import<<<(P.N + 255) / 256, 256, 0, s>>>(P, ctx->D, st);
        CK(cudaMemcpyAsync(ctx->D.part, part, sizeof(double4) * P.npart, cudaMemcpyDeviceToDevice, s));
        launch_body(ctx, s, 0, ctx->ghost_angle0, false);
    }
    return check_launch(ctx);
}

sph_status sph_step(sph_ctx* ctx, const float* u, int n_substeps, int ptr_on_device) {
    if (!ctx || !u || n_substeps < 0) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    cudaStream_t s = ctx->stream;
    const size_t ub = sizeof(float) * 3 * P.B;
    if (!ptr_on_device)
        for (int i = 0; i < 3 * P.B; ++i)
            if (!std::isfinite(u[i])) return fail(ctx, SPH_EINVAL, "non-finite input u");
    CK(cudaMemcpyAsync(ctx->D.u_cur, u, ub, ptr_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (ctx->exec == 3) {
        if (n_substeps > 0) CK(launch_resident(ctx, hold_args(ctx, n_substeps, 1.0f, 0)));
    } else if (ctx->coop) {
        if (n_substeps > 0) CK(launch_coop(ctx, n_substeps, 1.0f, 0));
    } else {
        for (int k = 0; k < n_substeps; ++k) launch_substep(ctx, 1.0f, 0);
    }
    sph_status st = check_launch(ctx);
    if (st) return st;
    if (!ptr_on_device) CK(cudaStreamSynchronize(s));
    return SPH_OK;
}

static sph_status accumulate_live(sph_ctx* ctx) {
    auto el = [&](const cudaEvent_t* ev, int a, int b, double* acc) -> cudaError_t {
        float m = 0.f;
        cudaError_t e = cudaEventElapsedTime(&m, ev[a], ev[b]);
        if (e == cudaSuccess) *acc += m;
        return e;
    };
    for (int q = 0; q < live_samples(ctx); ++q) {
        const cudaEvent_t* ev = ctx->live_ev.data() + (size_t)q * LIVE_SLOTS;
        CK(el(ev, LV_DEN0, LV_DEN1, &ctx->live_ms[SPH_LIVE_DENSITY]));
        if (ctx->small && ctx->fork && ctx->m2side) {
            // the two force launches overlap (main stream / rebuild branch): the force time of
            // the substep is the union of their active intervals
            double a = 0, b = 0, c = 0, d = 0;
            CK(el(ev, LV_SUB0, LV_F1_0, &a));
            CK(el(ev, LV_SUB0, LV_F1_1, &b));
            CK(el(ev, LV_SUB0, LV_F2_0, &c));
            CK(el(ev, LV_SUB0, LV_F2_1, &d));
            ctx->live_ms[SPH_LIVE_FORCE] += (b - a) + (d - c) - std::max(0.0, std::min(b, d) - std::max(a, c));
        } else {
            CK(el(ev, LV_F1_0, LV_F1_1, &ctx->live_ms[SPH_LIVE_FORCE]));
            if (ctx->small && ctx->fork) CK(el(ev, LV_F2_0, LV_F2_1, &ctx->live_ms[SPH_LIVE_FORCE]));
        }
        CK(el(ev, LV_SUB0, LV_SUB1, &ctx->live_ms[SPH_LIVE_SUBSTEP]));
        ++ctx->live_n;
    }
    return SPH_OK;
}

sph_status sph_set_live_timing(sph_ctx* ctx, int every) {
    if (!ctx || every < 0) return SPH_EINVAL;
    if (every == ctx->live_every) return SPH_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->tick_graph) {   // re-captured with (or without) the timing nodes on next use
        cudaGraphExecDestroy(ctx->tick_graph);
        ctx->tick_graph = nullptr;
    }
    for (auto e : ctx->live_ev) cudaEventDestroy(e);
    ctx->live_ev.clear();
    ctx->live_every = every;
    const size_t n = (size_t)live_samples(ctx) * LIVE_SLOTS;
    for (size_t q = 0; q < n; ++q) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ctx->live_ev.push_back(e);
    }
    for (double& m : ctx->live_ms) m = 0.0;
    ctx->live_n = 0;
    return SPH_OK;
}

sph_status sph_get_live_timing(sph_ctx* ctx, double* ms_sum, int64_t* n_samples, int reset) {
    if (!ctx || !ms_sum) return SPH_EINVAL;
    for (int t = 0; t < SPH_NUM_LIVE; ++t) ms_sum[t] = ctx->live_ms[t];
    if (n_samples) *n_samples = ctx->live_n;
    if (reset) {
        for (double& m : ctx->live_ms) m = 0.0;
        ctx->live_n = 0;
    }
    return SPH_OK;
}

static sph_status capture_tick_graph(sph_ctx* ctx) {
    if (ctx->tick_graph) return SPH_OK;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t ce = cudaSuccess;
    for (int k = 0; k < ctx->n_sub && ce == cudaSuccess; ++k) ce = launch_substep(ctx, 1.0f, 0, true, k);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
    if (ce != cudaSuccess) {
        if (e == cudaSuccess) cudaGraphDestroy(g);
        return fail(ctx, SPH_ECUDA, std::string("conditional node: ") + cudaGetErrorString(ce));
    }
    if (e != cudaSuccess) return fail(ctx, SPH_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&ctx->tick_graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        ctx->tick_graph = nullptr;
        return fail(ctx, SPH_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
    return SPH_OK;
}

sph_status sph_rollout_batch(sph_ctx* ctx, const float* u_seq, int K, const sph_pd_attitude* pd,
                             float* y_out, float* u_applied, int ptr_on_device) {
    if (!ctx || !u_seq || !y_out || K < 0) return SPH_EINVAL;
    if (pd && !pd->theta_ref) return fail(ctx, SPH_EINVAL, "pd->theta_ref is NULL");
    const DevParams& P = ctx->P;
    if (K == 0) return SPH_OK;
    cudaStream_t s = ctx->stream;
    const size_t nu = (size_t)P.B * K * 3, ny = (size_t)P.B * K * 6, nt = (size_t)P.B * K;
    const float *du = u_seq, *dth = pd ? pd->theta_ref : nullptr;
    float *dy = y_out, *dua = u_applied;
    if (!ptr_on_device) {   // stage host buffers through ctx-owned device memory
        for (size_t i = 0; i < nu; ++i)
            if (!std::isfinite(u_seq[i])) return fail(ctx, SPH_EINVAL, "non-finite input u");
        const size_t bytes = sizeof(float) * (nu + ny + nu + (pd ? nt : 0));
        sph_status st = ensure_stage(ctx, bytes);
        if (st) return st;
        float* base = (float*)ctx->stage;
        float* su = base;
        dy = base + nu;
        dua = u_applied ? base + nu + ny : nullptr;
        float* sth = base + nu + ny + nu;
        CK(cudaMemcpyAsync(su, u_seq, sizeof(float) * nu, cudaMemcpyHostToDevice, s));
        if (pd) CK(cudaMemcpyAsync(sth, pd->theta_ref, sizeof(float) * nt, cudaMemcpyHostToDevice, s));
        du = su;
        dth = pd ? sth : nullptr;
    }
    sph_status st = (ctx->coop || ctx->exec == 3) ? SPH_OK : capture_tick_graph(ctx);
    if (st) return st;
    const int tb = 128, tg = (P.B + tb - 1) / tb;
    for (int k = 0; k < K; ++k) {
        if (ctx->exec == 3) {   // sampling, ZOH / PD input and the n_sub substeps in one launch
            TickArgs T = hold_args(ctx, ctx->n_sub, 1.0f, 0);
            T.u_seq = du;
            T.theta_ref = dth;
            T.y = dy;
            T.u_applied = dua;
            T.K = K;
            T.k = k;
            T.pd = pd ? 1 : 0;
            T.Kp = pd ? pd->Kp : 0.0;
            T.Kd = pd ? pd->Kd : 0.0;
            CK(launch_resident(ctx, T));
            if (ctx->live_every > 0) {
                CK(cudaEventSynchronize(ctx->res_ev[1]));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, ctx->res_ev[0], ctx->res_ev[1]));
                ctx->live_ms[SPH_LIVE_TICK] += ms;
                ++ctx->live_n;
            }
            continue;
        }
        k_tick<<<tg, tb, 0, s>>>(P, ctx->D, du, dth, dy, dua, K, k, pd ? 1 : 0, pd ? pd->Kp : 0.0, pd ? pd->Kd : 0.0);
        if (ctx->coop) {
            CK(launch_coop(ctx, ctx->n_sub, 1.0f, 0));
            continue;
        }
        CK(cudaGraphLaunch(ctx->tick_graph, s));
        if (ctx->live_every > 0 && !ctx->coop) {   // read this tick's timing nodes before the next launch
            CK(cudaStreamSynchronize(s));
            st = accumulate_live(ctx);
            if (st) return st;
        }
    }
    st = check_launch(ctx);
    if (st) return st;
    if (!ptr_on_device) {
        CK(cudaMemcpyAsync(y_out, dy, sizeof(float) * ny, cudaMemcpyDeviceToHost, s));
        if (u_applied) CK(cudaMemcpyAsync(u_applied, dua, sizeof(float) * nu, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return all_failed(ctx);
    }
    return SPH_OK;
}

sph_status sph_get_body_state(sph_ctx* ctx, double* out) {
    if (!ctx || !out) return SPH_EINVAL;
    CK(cudaMemcpyAsync(out, ctx->D.body, 48 * (size_t)ctx->P.B, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
}

sph_status sph_settle(sph_ctx* ctx, double damping, int n_steps) {
    if (!ctx || n_steps < 0 || !(damping > 0 && damping <= 1)) return SPH_EINVAL;
    CK(cudaMemsetAsync(ctx->D.u_cur, 0, sizeof(float) * 3 * ctx->P.B, ctx->stream));
    if (ctx->exec == 3) {
        if (n_steps > 0) CK(launch_resident(ctx, hold_args(ctx, n_steps, (float)damping, 1)));
    } else if (ctx->coop) {
        if (n_steps > 0) CK(launch_coop(ctx, n_steps, (float)damping, 1));
    } else {
        for (int k = 0; k < n_steps; ++k) launch_substep(ctx, (float)damping, 1);
    }
    sph_status st = check_launch(ctx);
    if (st) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
}

sph_status sph_settle_until(sph_ctx* ctx, double damping, double v_tol, int max_steps,
                            int check_every, int* steps_done, float* max_speed) {
    if (!ctx || max_steps < 0 || check_every <= 0 || !(damping > 0 && damping <= 1) || !(v_tol >= 0))
        return SPH_EINVAL;
    const DevParams& P = ctx->P;
    sph_status st = ensure_stage(ctx, sizeof(float) * P.B);   // device [B] speeds
    if (st) return st;
    float* d_speed = static_cast<float*>(ctx->stage);
    std::vector<float> sp(P.B, 0.0f);
    int done = 0;
    // a spawn starts at rest, so the test runs after each chunk, never before the first one
    for (;;) {
        const int n = std::min(check_every, max_steps - done);
        if (n > 0) {
            st = sph_settle(ctx, damping, n);
            if (st) return st;
            done += n;
        }
        if (P.N > 0) {
            k_max_speed<<<P.B, 256, 0, ctx->stream>>>(P, ctx->D, d_speed);
            st = check_launch(ctx);
            if (st) return st;
            CK(cudaMemcpyAsync(sp.data(), d_speed, sizeof(float) * P.B, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        bool conv = true;
        for (float v : sp) conv = conv && v < v_tol;
        if (conv || done >= max_steps) break;
    }
    if (steps_done) *steps_done = done;
    if (max_speed) std::copy(sp.begin(), sp.end(), max_speed);
    return SPH_OK;
}

sph_status sph_get_status(sph_ctx* ctx, int32_t* rollout_status, int64_t* bad_step,
                          int32_t* bad_particle) {
    if (!ctx || !rollout_status) return SPH_EINVAL;
    std::vector<RolloutState> rs(ctx->P.B);
    CK(cudaMemcpyAsync(rs.data(), ctx->D.rs, sizeof(RolloutState) * ctx->P.B, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < ctx->P.B; ++b) {
        rollout_status[b] = rs[b].status;
        if (bad_step) bad_step[b] = rs[b].bad_step;
        if (bad_particle) bad_particle[b] = rs[b].bad_particle;
    }
    return SPH_OK;
}

sph_status sph_debug_cells(sph_ctx* ctx, int rollout, int32_t* cells, float* grid) {
    if (!ctx || !cells) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < 0 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    sph_status st = ensure_stage(ctx, sizeof(int) * 2 * std::max(P.N, 1));
    if (st) return st;
    k_debug_cells<<<(P.N + 255) / 256, 256, 0, ctx->stream>>>(P, ctx->D, rollout, (int*)ctx->stage);
    if ((st = check_launch(ctx))) return st;
    CK(cudaMemcpyAsync(cells, ctx->stage, sizeof(int) * 2 * P.N, cudaMemcpyDeviceToHost, ctx->stream));
    Geom gm;
    CK(cudaMemcpyAsync(&gm, ctx->D.geom + rollout, sizeof(Geom), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (grid) {
        volatile float rx = gm.rx, ry = gm.ry, hf = P.half;
        grid[0] = rx - hf;
        grid[1] = ry - hf;
        grid[2] = P.inv_C;
        grid[3] = P.C;
    }
    return SPH_OK;
}


sph_status sph_debug_neighbours(sph_ctx* ctx, int rollout, int64_t* nf_off, int32_t* nf_idx,
                                int64_t nf_cap, int64_t* g2_off, int32_t* g2_idx,
                                int64_t g2_cap, int64_t* g1_off, int32_t* g1_idx,
                                int64_t g1_cap) {
    if (!ctx || !nf_off || !g2_off || !g1_off) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < 0 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    cudaStream_t s = ctx->stream;
    if (!ctx->dbg_buf) CK(cudaMalloc(&ctx->dbg_buf, sizeof(int) * 3 * (size_t)std::max(P.N, 1) * (DBG_CAP + 1)));
    DevPtrs D = ctx->D;
    D.dbg_cnt = ctx->dbg_buf;
    D.dbg_idx = ctx->dbg_buf + 3 * (size_t)std::max(P.N, 1);
    // rebuild the cell list of the current state into the other buffer (state untouched)
    k_force_rebin<<<1, 1, 0, s>>>(ctx->D.rs, rollout);
    launch_rebin(ctx, s, true);
    if (P.N > 0) k_debug_neighbours<<<(P.N + 255) / 256, 256, 0, s>>>(P, D, rollout);
    sph_status st = check_launch(ctx);
    if (st) return st;
    std::vector<int> cnt(3 * (size_t)P.N), idx(3 * (size_t)P.N * DBG_CAP);
    if (P.N > 0) {
        CK(cudaMemcpyAsync(cnt.data(), D.dbg_cnt, sizeof(int) * cnt.size(), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(idx.data(), D.dbg_idx, sizeof(int) * idx.size(), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    int64_t* offs[3] = {nf_off, g2_off, g1_off};
    int32_t* outs[3] = {nf_idx, g2_idx, g1_idx};
    int64_t caps[3] = {nf_cap, g2_cap, g1_cap};
    for (int t = 0; t < 3; ++t) {
        int64_t tot = 0;
        offs[t][0] = 0;
        for (int i = 0; i < P.N; ++i) {
            const int n = cnt[(size_t)t * P.N + i];
            if (n > DBG_CAP) return fail(ctx, SPH_ENOMEM, "more than DBG_CAP neighbours");
            if (tot + n > caps[t]) return fail(ctx, SPH_ENOMEM, "neighbour cap too small");
            int* row = idx.data() + ((size_t)t * P.N + i) * DBG_CAP;
            std::sort(row, row + n);
            for (int q = 0; q < n; ++q) outs[t][tot + q] = row[q];
            tot += n;
            offs[t][i + 1] = tot;
        }
    }
    return SPH_OK;
}

sph_status sph_profile_substeps(sph_ctx* ctx, int n_substeps, float* ms) {
    if (!ctx || !ms || n_substeps < 1) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    cudaStream_t s = ctx->stream;
    if (ctx->exec == 3) {   // one resident launch of n_substeps (u held): ms per substep
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        cudaEventRecord(e0, s);
        CK(launch_resident(ctx, hold_args(ctx, n_substeps, 1.0f, 0)));
        cudaEventRecord(e1, s);
        CK(cudaEventSynchronize(e1));
        float m = 0.f;
        CK(cudaEventElapsedTime(&m, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        for (int t = 0; t < SPH_NUM_TIMERS; ++t) ms[t] = 0.f;
        ms[SPH_TIMER_SUBSTEP] = m / n_substeps;
        return SPH_OK;
    }
    cudaEvent_t ev[6];   // (ev[5]: between the sort and the lists of the rebuild timer)
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double acc[SPH_NUM_TIMERS] = {0};
    dim3 gp(P.ntile, P.B);
    // Sequential on the context stream (no fork), so every kernel is timed alone.  The rebuild
    // timer covers the plan + k_rebuild_small (small path; these also compute the rebuilt
    // rollouts' densities) or the eight rebuild kernels (multi-kernel path).
    for (int it = 0; it < n_substeps; ++it) {
        cudaEventRecord(ev[0], s);
        k_rebuild_plan<<<1, RB_T, 0, s>>>(P, ctx->D, 0, 0);
        if (ctx->small) k_rebuild_small<<<ctx->small_grid, RBS_T, ctx->small_smem, s>>>(P, ctx->D);
        else launch_rebin(ctx);
        cudaEventRecord(ev[5], s);
        launch_nlist_density(ctx, s);   // (runs after k_density in the step; same work)
        cudaEventRecord(ev[1], s);
        launch_density(ctx, s, 1);
        cudaEventRecord(ev[2], s);
        launch_force(ctx, s,1.0f);
        cudaEventRecord(ev[3], s);
        launch_body(ctx, s,0, ctx->ghost_angle0);
        cudaEventRecord(ev[4], s);
        sph_status st = check_launch(ctx);
        if (st) return st;
        CK(cudaEventSynchronize(ev[4]));
        for (int t = 0; t < 4; ++t) {
            float m;
            CK(cudaEventElapsedTime(&m, ev[t], ev[t + 1]));
            acc[t] += m;
        }
        float m;
        CK(cudaEventElapsedTime(&m, ev[0], ev[4]));
        acc[SPH_TIMER_SUBSTEP] += m;
        CK(cudaEventElapsedTime(&m, ev[0], ev[5]));
        acc[SPH_TIMER_SORT] += m;
    }
    for (int t = 0; t < SPH_NUM_TIMERS; ++t) ms[t] = (float)(acc[t] / n_substeps);
    for (auto& e : ev) cudaEventDestroy(e);
    return SPH_OK;
}

int sph_launches_per_substep(const sph_ctx* ctx) {
    // 0: one cooperative / resident launch per tick
    return ctx ? ((ctx->coop || ctx->exec == 3) ? 0 : launches_per_substep(ctx)) : 0;
}

int sph_launches_per_tick(const sph_ctx* ctx) {
    if (!ctx) return 0;
    if (ctx->exec == 3) return 1;
    if (ctx->coop) return 2;
    return 1 + ctx->n_sub * launches_per_substep(ctx);
}

int sph_exec_path(const sph_ctx* ctx, int* cluster_ctas, int* threads, int* slots_per_cta, int* smem_bytes) {
    if (!ctx) return 0;
    const bool r = ctx->exec == 3;
    if (cluster_ctas) *cluster_ctas = r ? ctx->res.CS : 0;
    if (threads) *threads = r ? ctx->res_nt : 0;
    if (slots_per_cta) *slots_per_cta = r ? ctx->res.S : 0;
    if (smem_bytes) *smem_bytes = r ? ctx->res.smem : 0;
    return ctx->exec;
}

sph_status sph_jacobian(sph_ctx* ctx, int rollout, double* A, double* B, int ptr_on_device) {
    if (!ctx || !A || !B) return SPH_EINVAL;
    const DevParams& P = ctx->P;
    if (rollout < 0 || rollout >= P.B) return fail(ctx, SPH_EINVAL, "rollout out of range");
    cudaStream_t s = ctx->stream;
    const int N = P.N, G = P.G, nx = 4 * N + 6, nd = nx + 3;
    JacParams J;
    J.N = N;
    J.G = G;
    J.nx = nx;
    J.h = ctx->fp.h;
    J.m = ctx->fp.mass;
    J.rho0 = ctx->fp.rho0;
    J.k = ctx->fp.k;
    J.clampP = ctx->fp.clamp_negative_pressure != 0.0 ? 1 : 0;
    J.gamma1 = ctx->fp.gamma1;
    J.alpha2h = 2.0 * ctx->fp.alpha * ctx->fp.h;
    J.beta = ctx->fp.beta;
    J.eps_h2 = ctx->fp.eps * ctx->fp.h * ctx->fp.h;
    J.m2 = ctx->fp.mass * ctx->fp.mass;
    J.sgn2m2 = ctx->fp.ghost_pressure_sign * 2.0 * J.m2;
    J.mB = ctx->bp.m;
    J.J = ctx->bp.J;
    J.H2 = 4.0 * J.h * J.h;
    J.h2 = J.h * J.h;
    J.wc = ctx->fp.w_cb_const;
    J.ws = 10.0 / M_PI;
    const size_t n1 = (size_t)std::max(N, 1), g1 = (size_t)std::max(G, 1);
    const int nblk = std::max(1, (N + JAC_T - 1) / JAC_T);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_pos = take(16 * n1), o_vel = take(16 * n1), o_body = take(48), o_gB = take(16 * g1),
                 o_gp = take(16 * g1), o_gv = take(16 * g1), o_ga = take(16 * g1),
                 o_nfc = take(4 * n1), o_nf = take(4 * n1 * JAC_NCAP), o_g2c = take(4 * n1),
                 o_g2 = take(4 * n1 * JAC_GCAP), o_g1c = take(4 * n1), o_g1 = take(4 * n1 * JAC_GCAP),
                 o_rho = take(8 * n1), o_P = take(8 * n1), o_Q = take(8 * n1),
                 o_hc = take(4 * n1), o_hop = take(4 * n1 * JAC_HCAP),
                 o_drho = take(8 * n1 * 9), o_ovf = take(4), o_bp = take(8 * 9 * 3 * (size_t)nblk),
                 o_A = ptr_on_device ? 0 : take(8 * (size_t)nx * nx), o_B = ptr_on_device ? 0 : take(24 * (size_t)nx);
    if (ctx->jac_bytes < off) {   // grow the cached scratch (kept for the next call)
        CK(cudaStreamSynchronize(s));
        if (ctx->jac_buf) cudaFree(ctx->jac_buf);
        ctx->jac_buf = nullptr;
        ctx->jac_bytes = 0;
        CK(cudaMalloc(&ctx->jac_buf, off));
        ctx->jac_bytes = off;
    }
    char* scratch = (char*)ctx->jac_buf;
    JacPtrs X;
    X.pos = (const double2*)(scratch + o_pos);
    X.vel = (const double2*)(scratch + o_vel);
    X.body = (const double*)(scratch + o_body);
    X.gB = (const double2*)(scratch + o_gB);
    X.gpos = (double2*)(scratch + o_gp);
    X.gvel = (double2*)(scratch + o_gv);
    X.garm = (double2*)(scratch + o_ga);
    X.nf_cnt = (int*)(scratch + o_nfc);
    X.nf = (int*)(scratch + o_nf);
    X.g2_cnt = (int*)(scratch + o_g2c);
    X.g2 = (int*)(scratch + o_g2);
    X.g1_cnt = (int*)(scratch + o_g1c);
    X.g1 = (int*)(scratch + o_g1);
    X.rho = (double*)(scratch + o_rho);
    X.P = (double*)(scratch + o_P);
    X.Q = (double*)(scratch + o_Q);
    X.hop_cnt = (int*)(scratch + o_hc);
    X.hop = (int*)(scratch + o_hop);
    X.drho = (double*)(scratch + o_drho);
    X.overflow = (int*)(scratch + o_ovf);
    X.bpart = (double*)(scratch + o_bp);
    double* dA = ptr_on_device ? A : (double*)(scratch + o_A);
    double* dB = ptr_on_device ? B : (double*)(scratch + o_B);
    X.A = dA;
    X.B = dB;
    cudaMemsetAsync(dA, 0, 8 * (size_t)nx * nx, s);   // A is sparse: seeds write only their rows
    cudaMemsetAsync(dB, 0, 24 * (size_t)nx, s);
    cudaMemsetAsync(X.overflow, 0, 4, s);
    if (G) cudaMemcpyAsync((void*)X.gB, ctx->D.ghost_b, 16 * (size_t)G, cudaMemcpyDeviceToDevice, s);
    k_jac_import<<<std::max(1, (std::max(N, 6) + 127) / 128), 128, 0, s>>>(
        P, ctx->D, rollout, (double2*)X.pos, (double2*)X.vel, (double*)X.body);
    if (G) k_jac_ghosts<<<(G + 127) / 128, 128, 0, s>>>(J, X);
    if (N) {
        k_jac_prep<<<(32 * N + 127) / 128, 128, 0, s>>>(J, X);   // one warp per particle
        k_jac_hops<<<(N + JAC_HOPS_WARPS - 1) / JAC_HOPS_WARPS, 32 * JAC_HOPS_WARPS,
                     sizeof(int) * JAC_HOPS_WARPS * JAC_CAND, s>>>(J, X);
    }
    // particle seeds (columns 0 .. 4N-1): one CTA each, writes its two-hop rows into A
    if (N) k_jac_pseed<<<4 * N, JAC_PT, 0, s>>>(J, X, 0);
    {   // body and input seeds (6 + 3 columns): every particle may respond, dense columns
        const int d0 = 4 * N, dc = 9;
        if (N) k_jac_drho<<<dim3((N + 127) / 128, dc), 128, 0, s>>>(J, X, d0);
        k_jac_col<<<dim3(nblk, dc), JAC_T, 0, s>>>(J, X, d0);
        k_jac_body<<<dc, 32, 0, s>>>(J, X, d0, nblk);
    }
    int ovf = 0;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&ovf, X.overflow, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && !ptr_on_device) {
        e = cudaMemcpyAsync(A, dA, 8 * (size_t)nx * nx, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(B, dB, 24 * (size_t)nx, cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(ctx, SPH_ECUDA, std::string("sph_jacobian: ") + cudaGetErrorString(e));
    if (ovf) return fail(ctx, SPH_ENOMEM, "sph_jacobian: more than 48 neighbours or ghosts, or 192 two-hop neighbours, of one particle");
    return SPH_OK;
}

sph_status sph_eigenvalues(sph_ctx* ctx, int n, double* A, double* w, int ptr_on_device) {
    if (!ctx || n < 1 || !A || !w) return SPH_EINVAL;
    cudaStream_t s = ctx->stream;
    if (!ctx->solver) {
        if (cusolverDnCreate(&ctx->solver) != CUSOLVER_STATUS_SUCCESS ||
            cusolverDnCreateParams(&ctx->solver_params) != CUSOLVER_STATUS_SUCCESS)
            return fail(ctx, SPH_ECUDA, "cuSOLVER handle creation failed");
    }
    cusolverDnSetStream(ctx->solver, s);
    const size_t An = (size_t)n * n;
    double* dA = A;
    double2* dW = nullptr;
    // scratch: [A copy if host] | W (complex) | device workspace
    size_t dws = 0, hws = 0;
    if (cusolverDnXgeev_bufferSize(ctx->solver, ctx->solver_params, CUSOLVER_EIG_MODE_NOVECTOR,
                                   CUSOLVER_EIG_MODE_NOVECTOR, n, CUDA_R_64F, dA, n, CUDA_C_64F,
                                   nullptr, CUDA_R_64F, nullptr, 1, CUDA_R_64F, nullptr, 1,
                                   CUDA_R_64F, &dws, &hws) != CUSOLVER_STATUS_SUCCESS)
        return fail(ctx, SPH_ECUDA, "cusolverDnXgeev_bufferSize failed");
    const size_t oA = 0, oW = ptr_on_device ? 0 : ((8 * An + 255) & ~(size_t)255);
    const size_t oWs = oW + ((16 * (size_t)n + 255) & ~(size_t)255), need = oWs + dws + 16;
    if (ctx->eig_dbytes < need) {
        CK(cudaStreamSynchronize(s));
        if (ctx->eig_dbuf) cudaFree(ctx->eig_dbuf);
        ctx->eig_dbuf = nullptr;
        ctx->eig_dbytes = 0;
        CK(cudaMalloc(&ctx->eig_dbuf, need));
        ctx->eig_dbytes = need;
    }
    if (ctx->eig_hbuf.size() < hws + 16) ctx->eig_hbuf.resize(hws + 16);
    char* base = (char*)ctx->eig_dbuf;
    if (!ptr_on_device) {
        dA = (double*)(base + oA);
        CK(cudaMemcpyAsync(dA, A, 8 * An, cudaMemcpyHostToDevice, s));
    }
    dW = ptr_on_device ? (double2*)w : (double2*)(base + oW);
    int* dinfo = (int*)(base + oWs + dws);
    if (cusolverDnXgeev(ctx->solver, ctx->solver_params, CUSOLVER_EIG_MODE_NOVECTOR,
                        CUSOLVER_EIG_MODE_NOVECTOR, n, CUDA_R_64F, dA, n, CUDA_C_64F, dW, CUDA_R_64F,
                        nullptr, 1, CUDA_R_64F, nullptr, 1, CUDA_R_64F, base + oWs, dws,
                        ctx->eig_hbuf.data(), hws, dinfo) != CUSOLVER_STATUS_SUCCESS)
        return fail(ctx, SPH_ECUDA, "cusolverDnXgeev failed");
    int info = 0;
    CK(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (!ptr_on_device) CK(cudaMemcpyAsync(w, dW, 16 * (size_t)n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (info != 0) return fail(ctx, SPH_ECUDA, "cusolverDnXgeev: info = " + std::to_string(info));
    return SPH_OK;
}

sph_status sph_get_counters(sph_ctx* ctx, int64_t* steps, int32_t* rebuilds) {
    if (!ctx) return SPH_EINVAL;
    std::vector<RolloutState> rs(ctx->P.B);
    CK(cudaMemcpyAsync(rs.data(), ctx->D.rs, sizeof(RolloutState) * ctx->P.B, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < ctx->P.B; ++b) {
        if (steps) steps[b] = rs[b].step;
        if (rebuilds) rebuilds[b] = rs[b].rebuilds;
    }
    return SPH_OK;
}

void sph_get_sizes(const sph_ctx* ctx, int* n_fluid, int* n_ghost, int* n_rollouts, int* n_cells) {
    if (!ctx) return;
    if (n_fluid) *n_fluid = ctx->P.N;
    if (n_ghost) *n_ghost = ctx->P.G;
    if (n_rollouts) *n_rollouts = ctx->P.B;
    if (n_cells) *n_cells = ctx->P.ncell;
}

const char* sph_last_error(const sph_ctx* ctx) { return ctx ? ctx->err.c_str() : g_init_err.c_str(); }

void sph_destroy(sph_ctx* ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->tick_graph) cudaGraphExecDestroy(ctx->tick_graph);
    if (ctx->stage) cudaFree(ctx->stage);
    if (ctx->dbg_buf) cudaFree(ctx->dbg_buf);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->side2) cudaStreamDestroy(ctx->side2);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    for (auto e : ctx->live_ev) cudaEventDestroy(e);
    for (auto e : ctx->res_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->jac_buf) cudaFree(ctx->jac_buf);
    if (ctx->g1_buf) cudaFree(ctx->g1_buf);
    if (ctx->eig_dbuf) cudaFree(ctx->eig_dbuf);
    if (ctx->solver_params) cusolverDnDestroyParams(ctx->solver_params);
    if (ctx->solver) cusolverDnDestroy(ctx->solver);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

}  // extern "C"
