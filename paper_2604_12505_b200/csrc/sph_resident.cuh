// sph_resident.cuh -- rollout-resident slow tick (exec_path 3): one thread-block CLUSTER per
// rollout keeps the rollout's particles in distributed shared memory for a whole slow tick
// (n_sub substeps of Algorithm 1, + symplectic Euler, inside the multi-rate
// loop of P:263 / P:325).  Global memory is touched once per tick (state in / out, y_k, u_k).
//
// Partition.  The rollout's particles are kept sorted by the composite key (cell, canonical id)
// (cells row-major, side 2h + skin, reading A19 / A20).  CTA r of the cluster owns the global
// sorted slots [r S, r S + n_own), S a multiple of 32 (so a warp's 32 slots are the same 32-slot
// group in every cluster shape and the per-warp body partials do not depend on CS).
// Each CTA holds a WINDOW: its own slots plus the halo slots of the neighbouring CTAs that its
// particles' 3 x 3 cell blocks reach, at window index HCAP + (g - r S) for global slot g.
// Window cell table wcs[c - cbase] = first window index whose cell is >= c, so a particle's
// fluid candidates are three contiguous window ranges (cell rows cy-1..cy+1, cells cx-1..cx+1).
//
// Substep (all CTAs of the cluster):
//   [rebuild when the Verlet bound tripped: cell keys -> distributed merge sort (particles whose
//    cell is unchanged stay a sorted subsequence; the few "movers" are ranked globally) ->
//    scatter to the new owners -> window + halo pull -> cell table -> Verlet lists]
//   density + EOS of own slots (Eq. density_update, Eq. EOS)
//   cluster barrier A; pull the halo's (rho, P/rho^2)
//   forces, wall, kick-drift of own slots (Eqs. momentum, viscous P:145-163, pressure_b2f,
//     viscous_b2f P:188-203, Alg. 1 l.8 P:248); per-warp body partials to every CTA
//   cluster barrier B; pull the halo's new state
//   body: fixed-order fp64 reduction of all warp partials (every CTA, identical bits),
//     Eq. tankdynamics, kick-drift, Eq. kinematicghost into shared memory
// Every result depends only on the rollout (no atomics on any value path): bitwise independent of
// the batch, of the rollout's position in it and of the cluster size.
#pragma once
#include "sph_kernels.cuh"

namespace sph {

constexpr int RES_MAXT = 640;    // threads per CTA (upper bound; 20 warps)
constexpr int RES_RU = 4;        // own slots per thread in the rebuild phases (S <= RES_RU * NT)
constexpr int RES_MAXCS = 16;    // cluster size bound (8 portable, 16 non-portable)

struct ResParams {
    int CS, S, HCAP, W, KR, KQ, IDB, MCAP, NCT, npart;
    uint32_t idmask;
    // dynamic shared memory carve-up (byte offsets, 16-byte aligned)
    int o_pv, o_rpv, o_gst, o_glo, o_ghb, o_part, o_aux, o_xb, o_nbr, o_key, o_rkey, o_nmk, o_obk, o_mkg,
        o_mks, o_wcs, o_obj, o_ncnt, o_misc;
    int smem;
};

// per-tick arguments (u_seq == nullptr: hold D.u_cur, no sampling -- sph_step / sph_settle)
struct TickArgs {
    const float* u_seq;
    const float* theta_ref;
    float* y;
    float* u_applied;
    int K, k, pd;
    double Kp, Kd;
    int n_sub;
    float damping;
    int pin;
    float ghost_angle0;
    unsigned long long* clk;   // diagnostic build only (SPH_RES_TIMING); nullptr otherwise
};

struct ResMisc {
    double body[8];          // r_x r_y theta rd_x rd_y thd | cos theta, sin theta
    float u[3];
    float rbx, rby;          // body position (float) at the last rebuild (Verlet criterion)
    float disp;
    float skin, rl2, rdisp;  // adaptive Verlet skin of the current lists (B5)
    long long last_reb;
    int need_rebin, stop, n_reb, it_done;
    int wlo, whi, cbase, cend;
    int nm, mv;              // this CTA's non-mover / mover counts (read by the other CTAs)
    uint32_t nm_min, nm_max;
    int unsorted;
    int M;
    int bad_all[RES_MAXCS];  // sticky status flags of the cluster's CTAs (written remotely)
    int nm_all[RES_MAXCS], mv_all[RES_MAXCS], nmpre[RES_MAXCS + 1], mvpre[RES_MAXCS + 1];
    uint32_t mn_all[RES_MAXCS], mx_all[RES_MAXCS];
    int wt[32];              // block-scan scratch
};

// ---------------------------------------------------------------------------------------
// cluster helpers (sm_90+ PTX)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
}
// full cluster barrier: every thread of every CTA arrives (release) and waits (acquire), so the
// shared-memory stores of all CTAs before it are visible to all CTAs after it
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// generic address of the same shared-memory object in CTA `rank` of the cluster (DSMEM)
template <class T>
__device__ __forceinline__ T* cl_map(T* p, int rank) {
    uint64_t out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"((uint64_t)p), "r"(rank));
    return reinterpret_cast<T*>(out);
}

// Phase timestamps of a diagnostic build (-DSPH_RES_TIMING): thread 0 of every CTA records
// %globaltimer at RES_NMARK points of each substep into TickArgs::clk [cta][substep][RES_NMARK]
// (nanoseconds): 0 start, 1 after rebuild, 2 after density, 3 after barrier A, 4 after aux pull +
// forces, 5 after barrier B, 6 after the partial loads (warp 0), 7 after the warp reduction,
// 8 after the body update (lane 0), 9 after the pv pull (block barrier), 10 after the ghosts.
// RES_MARKD: the same, ordered after the computation of the double v (a register dependency).
// The stamps perturb the code they bracket: the diagnostic build runs a C2 substep in 14.0 us
// against 9.3 us without them, 4.5 us of it in warp 0's fp64 butterfly right after a stamp store
// (a shared-memory reduction there brings the build to 9.9 us; the product build is slower with
// it) -- read phase SHARES and per-CTA spreads from it, not absolute times.
constexpr int RES_NMARK = 11;
#ifdef SPH_RES_TIMING
#define RES_MARK(T_, ph_, it_)                                                                    \
    do {                                                                                         \
        if (threadIdx.x == 0 && (T_).clk) {                                                      \
            unsigned long long t_;                                                               \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
            (T_).clk[((size_t)blockIdx.x * (T_).n_sub + (it_)) * RES_NMARK + (ph_)] = t_;        \
        }                                                                                        \
    } while (0)
#define RES_MARKD(T_, ph_, it_, v_)                                                               \
    do {                                                                                         \
        if (threadIdx.x == 0 && (T_).clk) {                                                      \
            unsigned long long t_;                                                               \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "d"(v_));                     \
            (T_).clk[((size_t)blockIdx.x * (T_).n_sub + (it_)) * RES_NMARK + (ph_)] = t_;        \
        }                                                                                        \
    } while (0)
#else
#define RES_MARK(T_, ph_, it_) do { } while (0)
#define RES_MARKD(T_, ph_, it_, v_) do { } while (0)
#endif

__device__ __forceinline__ void set_status_at(RolloutState* rs, int code, int particle, long long step) {
    if (atomicCAS(&rs->status, 0, code) == 0) {
        rs->bad_step = step;
        rs->bad_particle = particle;
    }
}

// exclusive block scan of one int per thread (blockDim.x <= 1024); wt: >= 32 ints of smem
__device__ __forceinline__ int res_scan(int v, int* total, int* wt) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wt[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = lane < nw ? wt[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, d);
            if (lane >= d) t += y;
        }
        if (lane < nw) wt[lane] = t;
    }
    __syncthreads();
    const int base = w ? wt[w - 1] : 0;
    *total = wt[nw - 1];
    __syncthreads();
    return base + x - v;
}

__device__ __forceinline__ int lower_bound_u32(const uint32_t* a, int n, uint32_t k) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (a[m] < k) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// ---------------------------------------------------------------------------------------
// The shared-memory view of one CTA
// ---------------------------------------------------------------------------------------
struct ResSmem {
    float4* pv;        // [W] window state (x, y, vx, vy)
    float4* rpv;       // [S] receive buffer: sorted state after a rebuild's scatter; new state
                       //     written by the force pass (the halo of the other CTAs pulls it)
    float4* gst;       // [G] ghost world state (x_hi, y_hi, vx, vy)
    float4* glo;       // [G] (x_lo, y_lo, arm_x, arm_y)
    double2* ghb;      // [G] body-frame ghost positions (constant; copied once per launch)
    double4* part;     // [npart] per-warp body partials of the whole rollout (written remotely)
    float2* aux;       // [W] (rho, P / rho^2)
    float2* xb;        // [S] own positions at the last rebuild
    uint2* nbr;        // [KQ][S] Verlet lists: window indices (u16), four per uint2
    uint32_t* key;     // [W] composite key (cell << IDB | id) of the window slots
    uint32_t* rkey;    // [S] receive buffer keys
    uint32_t* nmk;     // [S] keys of own non-movers (sorted; read remotely)
    uint32_t* obk;     // [S] keys of own movers (read remotely)
    uint32_t* mkg;     // [MCAP] gathered mover keys
    uint32_t* mks;     // [MCAP] gathered mover keys, sorted
    uint16_t* wcs;     // [NCT] window cell table
    uint16_t* obj;     // [S] own slot of each own mover
    uint8_t* ncnt;     // [S] list length (NL_OVERFLOW: cell scan)
    ResMisc* m;
};

__device__ __forceinline__ ResSmem res_smem(const ResParams& R, unsigned char* base) {
    ResSmem s;
    s.pv = reinterpret_cast<float4*>(base + R.o_pv);
    s.rpv = reinterpret_cast<float4*>(base + R.o_rpv);
    s.gst = reinterpret_cast<float4*>(base + R.o_gst);
    s.glo = reinterpret_cast<float4*>(base + R.o_glo);
    s.ghb = reinterpret_cast<double2*>(base + R.o_ghb);
    s.part = reinterpret_cast<double4*>(base + R.o_part);
    s.aux = reinterpret_cast<float2*>(base + R.o_aux);
    s.xb = reinterpret_cast<float2*>(base + R.o_xb);
    s.nbr = reinterpret_cast<uint2*>(base + R.o_nbr);
    s.key = reinterpret_cast<uint32_t*>(base + R.o_key);
    s.rkey = reinterpret_cast<uint32_t*>(base + R.o_rkey);
    s.nmk = reinterpret_cast<uint32_t*>(base + R.o_nmk);
    s.obk = reinterpret_cast<uint32_t*>(base + R.o_obk);
    s.mkg = reinterpret_cast<uint32_t*>(base + R.o_mkg);
    s.mks = reinterpret_cast<uint32_t*>(base + R.o_mks);
    s.wcs = reinterpret_cast<uint16_t*>(base + R.o_wcs);
    s.obj = reinterpret_cast<uint16_t*>(base + R.o_obj);
    s.ncnt = reinterpret_cast<uint8_t*>(base + R.o_ncnt);
    s.m = reinterpret_cast<ResMisc*>(base + R.o_misc);
    return s;
}

// float pose of the body state in shared memory (the particle kernels' Geom)
__device__ __forceinline__ Geom res_geom(const ResMisc* m, float ghost_angle0) {
    return Geom{(float)m->body[0], (float)m->body[1], (float)(m->body[2] + ghost_angle0),
                (float)m->body[3], (float)m->body[4], {0.f, 0.f, 0.f}};
}

// Eq. kinematicghost in fp64 for every ghost, into shared memory (hi/lo split B2)
__device__ __forceinline__ void res_ghosts(const DevParams& P, const DevPtrs& D, const ResSmem& s) {
    const double* bd = s.m->body;
    const double c = bd[6], sn = bd[7], r0 = bd[0], r1 = bd[1], v0 = bd[3], v1 = bd[4], w = bd[5];
    for (int g = threadIdx.x; g < P.G; g += blockDim.x) {
        const double2 q = s.ghb[g];
        const double ax = c * q.x - sn * q.y, ay = sn * q.x + c * q.y;
        const double wx = ax + r0, wy = ay + r1;
        const double vx = v0 - w * (wy - r1);
        const double vy = v1 + w * (wx - r0);
        const float hx = (float)wx, hy = (float)wy;
        s.gst[g] = make_float4(hx, hy, (float)vx, (float)vy);
        s.glo[g] = make_float4((float)(wx - (double)hx), (float)(wy - (double)hy), (float)(wx - r0),
                               (float)(wy - r1));
    }
}

// ---------------------------------------------------------------------------------------
// Rebuild: distributed merge sort by (cell, id), window, halo, cell table, Verlet lists
// ---------------------------------------------------------------------------------------
__device__ __noinline__ void res_sort(const DevParams& P, const ResParams& R, const ResSmem& s,
                                      RolloutState* rs, int r, int lo, int n_own, long long step) {
    ResMisc* m = s.m;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int hi = lo + n_own;
    // R1: new composite keys of own slots (contiguous chunk per thread, so block scans keep the
    // slot order); movers = slots whose cell changed since the last rebuild
    const float rx = (float)m->body[0], ry = (float)m->body[1];
    const float ox = __fsub_rn(rx, P.half), oy = __fsub_rn(ry, P.half);
    uint32_t nk[RES_RU];
    int mov[RES_RU];
    const int j0 = tid * RES_RU;
    int cnm = 0, cmv = 0;
#pragma unroll
    for (int e = 0; e < RES_RU; ++e) {
        const int j = j0 + e;
        nk[e] = 0u;
        mov[e] = 0;
        if (j < n_own) {
            const float4 x = s.pv[R.HCAP + j];
            const uint32_t ok = s.key[R.HCAP + j];
            int cx = cell_coord(x.x, ox, P.inv_C), cy = cell_coord(x.y, oy, P.inv_C);
            if (cx < 1 || cx > P.nx - 2 || cy < 1 || cy > P.nx - 2) {   // tunnelled out of the tank
                set_status_at(rs, 3, (int)(ok & R.idmask), step);
                for (int t = 0; t < R.CS; ++t) cl_map(m->bad_all + r, t)[0] = 3;
                cx = min(max(cx, 1), P.nx - 2);
                cy = min(max(cy, 1), P.nx - 2);
            }
            nk[e] = ((uint32_t)(cy * P.nx + cx) << R.IDB) | (ok & R.idmask);
            mov[e] = nk[e] != ok;
            cnm += !mov[e];
            cmv += mov[e];
        }
    }
    // R2: compaction (non-mover keys stay sorted: the old keys were)
    int nm, mv;
    int a0 = res_scan(cnm, &nm, m->wt);
    int m0 = res_scan(cmv, &mv, m->wt);
    if (tid == 0) m->unsorted = 0;
#pragma unroll
    for (int e = 0; e < RES_RU; ++e) {
        const int j = j0 + e;
        if (j >= n_own) break;
        if (!mov[e]) s.nmk[a0++] = nk[e];
        else {
            s.obk[m0] = nk[e];
            s.obj[m0++] = (uint16_t)j;
        }
    }
    __syncthreads();
    for (int a = tid + 1; a < nm; a += NT)
        if (s.nmk[a - 1] >= s.nmk[a]) m->unsorted = 1;
    __syncthreads();
    if (m->unsorted) {   // not a sorted start: every slot is a mover (CTA-uniform)
        nm = 0;
        mv = n_own;
#pragma unroll
        for (int e = 0; e < RES_RU; ++e) {
            const int j = j0 + e;
            if (j < n_own) {
                s.obk[j] = nk[e];
                s.obj[j] = (uint16_t)j;
                mov[e] = 1;
            }
        }
    }
    // this CTA's movers / non-movers for the other CTAs
    if (tid == 0) {
        m->nm = nm;
        m->mv = mv;
        m->nm_min = nm ? s.nmk[0] : 0xffffffffu;
        m->nm_max = nm ? s.nmk[nm - 1] : 0u;
    }
    // non-mover index of each own non-mover (recomputed from the scan position)
    int anm[RES_RU];
    {
        int a = nm ? a0 - cnm : 0;   // a0 was advanced by cnm above
#pragma unroll
        for (int e = 0; e < RES_RU; ++e) {
            anm[e] = a;
            if (j0 + e < n_own && !mov[e]) ++a;
        }
    }
    cl_sync();   // #1: counts, non-mover and mover keys of every CTA visible
    if (tid < R.CS) {
        const ResMisc* mr = cl_map(m, tid);
        m->nm_all[tid] = mr->nm;
        m->mv_all[tid] = mr->mv;
        m->mn_all[tid] = mr->nm_min;
        m->mx_all[tid] = mr->nm_max;
    }
    __syncthreads();
    if (tid == 0) {
        int a = 0, b = 0;
        for (int t = 0; t < R.CS; ++t) {
            m->nmpre[t] = a;
            m->mvpre[t] = b;
            a += m->nm_all[t];
            b += m->mv_all[t];
        }
        m->nmpre[R.CS] = a;
        m->mvpre[R.CS] = b;
        m->M = b;
    }
    __syncthreads();
    const int M = m->M;
    // R4: number of movers (cluster-wide) with a smaller key than each own slot's new key
    auto mover_key = [&](int gi) {
        int o = 0;
        while (m->mvpre[o + 1] <= gi) ++o;
        return cl_map(s.obk, o)[gi - m->mvpre[o]];
    };
    int cntM[RES_RU];
#pragma unroll
    for (int e = 0; e < RES_RU; ++e) cntM[e] = 0;
    if (M <= R.MCAP) {
        for (int gi = tid; gi < M; gi += NT) s.mkg[gi] = mover_key(gi);
        __syncthreads();
        for (int gi = tid; gi < M; gi += NT) {   // rank by counting (keys are unique)
            const uint32_t k = s.mkg[gi];
            int rank = 0;
            for (int x = 0; x < M; ++x) rank += s.mkg[x] < k;
            s.mks[rank] = k;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < RES_RU; ++e)
            if (j0 + e < n_own) cntM[e] = lower_bound_u32(s.mks, M, nk[e]);
    } else {   // many movers (unsorted start): chunked counting
        for (int c0 = 0; c0 < M; c0 += R.MCAP) {
            const int cn = min(R.MCAP, M - c0);
            for (int gi = tid; gi < cn; gi += NT) s.mkg[gi] = mover_key(c0 + gi);
            __syncthreads();
#pragma unroll
            for (int e = 0; e < RES_RU; ++e) {
                if (j0 + e >= n_own) continue;
                int c = 0;
                for (int x = 0; x < cn; ++x) c += s.mkg[x] < nk[e];
                cntM[e] += c;
            }
            __syncthreads();
        }
    }
    // R5 + R6: new global slot of every own slot, scatter to its owner's receive buffer
#pragma unroll
    for (int e = 0; e < RES_RU; ++e) {
        const int j = j0 + e;
        if (j >= n_own) continue;
        int g;
        if (!mov[e]) {
            g = m->nmpre[r] + anm[e] + cntM[e];
        } else {
            g = cntM[e];
            for (int t = 0; t < R.CS; ++t) {
                const int n = m->nm_all[t];
                if (n == 0 || nk[e] < m->mn_all[t]) continue;
                if (nk[e] > m->mx_all[t]) {
                    g += n;
                    continue;
                }
                g += lower_bound_u32(t == r ? s.nmk : cl_map(s.nmk, t), n, nk[e]);
            }
        }
        const int o = g / R.S, t = g - o * R.S;
        cl_map(s.rpv, o)[t] = s.pv[R.HCAP + j];
        cl_map(s.rkey, o)[t] = nk[e];
    }
    cl_sync();   // #2: every CTA's receive buffer holds its new sorted own slots
}

// R7 + R8 (after every CTA's receive buffer rpv / rkey holds its sorted own slots): window
// [wlo, whi) = the global slots in cells [c_first - nx - 1, c_last + nx + 2), halo pull, window
// cell table, Verlet lists.  FROM_XB = false (rebuild): the lists and xb come from the current
// positions.  FROM_XB = true (tick-start reload of the lists of the last rebuild): every CTA has
// put its own rebuild-time positions xb into aux[HCAP + j]; the lists are rebuilt from xb of the
// window, i.e. exactly the lists of that rebuild (same cells, same positions, same predicate).
template <bool FROM_XB>
__device__ __noinline__ void res_window(const DevParams& P, const ResParams& R, const ResSmem& s,
                                        RolloutState* rs, int r, int lo, int n_own, long long step) {
    ResMisc* m = s.m;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int hi = lo + n_own;
    if (tid == 0 || tid == 32) {
        const bool low = tid == 0;
        const uint32_t c = low ? (s.rkey[0] >> R.IDB) - (uint32_t)P.nx - 1u
                               : (s.rkey[n_own - 1] >> R.IDB) + (uint32_t)P.nx + 2u;
        const uint32_t target = c << R.IDB;
        int a = low ? 0 : hi, b = low ? lo : P.N;
        while (a < b) {
            const int mid = (a + b) >> 1;
            const int o = mid / R.S;
            const uint32_t k = cl_map(s.rkey, o)[mid - o * R.S];
            if (k < target) a = mid + 1;
            else b = mid;
        }
        if (low) {
            if (lo - a > R.HCAP) {   // halo larger than the window capacity
                set_status_at(rs, 4, -1, step);
                for (int t = 0; t < R.CS; ++t) cl_map(m->bad_all + r, t)[0] = 4;
                a = lo - R.HCAP;
            }
            m->wlo = a;
            m->cbase = (int)c;
        } else {
            if (a - hi > R.HCAP) {
                set_status_at(rs, 4, -1, step);
                for (int t = 0; t < R.CS; ++t) cl_map(m->bad_all + r, t)[0] = 4;
                a = hi + R.HCAP;
            }
            m->whi = a;
            m->cend = (int)c;
        }
    }
    for (int j = tid; j < n_own; j += NT) {
        s.pv[R.HCAP + j] = s.rpv[j];
        s.key[R.HCAP + j] = s.rkey[j];
    }
    __syncthreads();
    const int wlo = m->wlo, whi = m->whi, nlow = lo - wlo, nhigh = whi - hi;
    for (int q = tid; q < nlow + nhigh; q += NT) {
        const int g = q < nlow ? wlo + q : hi + (q - nlow);
        const int o = g / R.S, t = g - o * R.S;
        s.pv[R.HCAP + (g - lo)] = cl_map(s.rpv, o)[t];
        s.key[R.HCAP + (g - lo)] = cl_map(s.rkey, o)[t];
        if (FROM_XB) s.aux[R.HCAP + (g - lo)] = cl_map(s.aux, o)[R.HCAP + t];
    }
    __syncthreads();
    // R8: window cell table
    const int wl = R.HCAP - nlow, wh = R.HCAP + n_own + nhigh;
    const int cbase = m->cbase, cend = m->cend;
    for (int w = wl + tid; w < wh; w += NT) {
        const int c = (int)(s.key[w] >> R.IDB);
        const int cp = w == wl ? cbase - 1 : (int)(s.key[w - 1] >> R.IDB);
        for (int cc = max(cp + 1, cbase); cc <= min(c, cend); ++cc) s.wcs[cc - cbase] = (uint16_t)w;
    }
    if (tid == 0) {
        const int cl = wh > wl ? (int)(s.key[wh - 1] >> R.IDB) : cbase - 1;
        for (int cc = max(cl + 1, cbase); cc <= cend; ++cc) s.wcs[cc - cbase] = (uint16_t)wh;
        if (!FROM_XB) {
            m->rbx = (float)m->body[0];
            m->rby = (float)m->body[1];
            m->n_reb += 1;
        }
        m->need_rebin = 0;
    }
    __syncthreads();
    // window positions of the list predicate: current state (rebuild) or rebuild-time xb (reload)
    const float2* __restrict__ wpos = FROM_XB ? s.aux : reinterpret_cast<const float2*>(s.pv);
    const float RL2 = m->rl2;   // list radius^2 of these lists (adaptive skin, B5)
    const int ws = FROM_XB ? 1 : 2;
    // Verlet lists of own slots: every window slot of the 3 x 3 cell block within 2h + skin
    // (canonical float32 predicate, reading A19), ascending window index; the partial last quad
    // is padded with the slot itself (exact zero force, W(0) subtracted in the density)
    for (int j = tid; j < n_own; j += NT) {
        const int li = R.HCAP + j;
        const float2 xi = wpos[ws * li];
        const int c = (int)(s.key[li] >> R.IDB);
        uint2* nq = s.nbr + j;
        int n = 0;
        bool ovf = false;
        uint64_t acc = 0;
        for (int dy = -1; dy <= 1; ++dy) {
            const int c0 = c + dy * P.nx - 1 - cbase;
            const int w0 = s.wcs[c0], w1 = s.wcs[c0 + 3];
            for (int w = w0; w < w1; ++w) {
                if (w == li) continue;
                const float2 xj = wpos[ws * w];
                if (dist2(__fsub_rn(xi.x, xj.x), __fsub_rn(xi.y, xj.y)) < RL2) {
                    if (n >= R.KR) {
                        ovf = true;
                        continue;
                    }
                    acc = (acc >> 16) | ((uint64_t)(uint16_t)w << 48);
                    if ((++n & 3) == 0) {
                        *nq = make_uint2((uint32_t)acc, (uint32_t)(acc >> 32));
                        nq += R.S;
                    }
                }
            }
        }
        if (!ovf && (n & 3)) {
            const int pad = 4 - (n & 3);
            for (int t = 0; t < pad; ++t) acc = (acc >> 16) | ((uint64_t)(uint16_t)li << 48);
            *nq = make_uint2((uint32_t)acc, (uint32_t)(acc >> 32));
        }
        s.ncnt[j] = (uint8_t)(ovf ? NL_OVERFLOW : n);
        s.xb[j] = xi;
    }
    __syncthreads();
}

// Full rebuild of a substep: sort (R1-R6), then window, halo, cell table and lists.
__device__ __forceinline__ void res_rebuild(const DevParams& P, const ResParams& R, const ResSmem& s,
                                            RolloutState* rs, int r, int lo, int n_own, long long step) {
    res_sort(P, R, s, rs, r, lo, n_own, step);
    res_window<false>(P, R, s, rs, r, lo, n_own, step);
}

// window index of the t-th entry of a quad (u16)
__device__ __forceinline__ int quad_idx(uint2 w, int t) {
    const uint32_t h = (t & 2) ? w.y : w.x;
    return (t & 1) ? (int)(h >> 16) : (int)(h & 0xffffu);
}

// three candidate window ranges of the cell block of window slot li (list overflow fallback)
template <class F>
__device__ __forceinline__ void res_cell_candidates(const DevParams& P, const ResParams& R,
                                                    const ResSmem& s, int li, F&& f) {
    const int c = (int)(s.key[li] >> R.IDB) - s.m->cbase;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
        const int c0 = c + dy * P.nx - 1;
        const int w0 = s.wcs[c0], w1 = s.wcs[c0 + 3];
        for (int w = w0; w < w1; ++w) f(w);
    }
}

// Density + EOS of own slot j (window index li): Eq. density_update, Eq. EOS (see density_core)
__device__ __forceinline__ void res_density(const DevParams& P, const ResParams& R, const ResSmem& s,
                                            const Geom& gm, int j) {
    const int li = R.HCAP + j;
    const float4 x4 = s.pv[li];
    const float2 p = make_float2(x4.x, x4.y);
    float wf = 4.0f;   // self term W_cb(0) ("all particles")
    const int n = s.ncnt[j];
    const float2* __restrict__ p2 = reinterpret_cast<const float2*>(s.pv);
    auto pos = [&](int w) { return p2[2 * w]; };   // (x, y) half of the state: one 8-byte load
    if (n != NL_OVERFLOW) {
        const uint2* nq = s.nbr + j;
        uint2 wn = *nq;
        for (int k = 0; k < n; k += 4) {
            const uint2 w = wn;
            nq += R.S;
            if (k + 4 < n) wn = *nq;
            wf += w_list2(P, p, pos(quad_idx(w, 0)), pos(quad_idx(w, 1)));
            if (k + 2 < n) wf += w_list2(P, p, pos(quad_idx(w, 2)), pos(quad_idx(w, 3)));
        }
        wf -= 4.0f * (float)(((n + 1) & ~1) - n);   // padding entries (self) added W(0) = 4 each
    } else {
        res_cell_candidates(P, R, s, li, [&](int w) { wf += w_masked(P, x4, s.pv[w], w != li); });
    }
    float wg = 0.0f;
    for_ghost_candidates(P, gm, p, P.ghost_K, P.wall_r2, [&](int g) {
        const float4 xg = s.gst[g];
        const float dx = __fsub_rn(p.x, xg.x), dy = __fsub_rn(p.y, xg.y);
        if (dist2(dx, dy) < P.H2) {
            const float4 lo = s.glo[g];
            const float ex = dx - lo.x, ey = dy - lo.y;
            const float r2 = ex * ex + ey * ey;
            wg += wcb_poly(r2 > 0.0f ? r2 * rsqrtf(r2) * P.inv_h : 0.0f);
        }
    });
    const float rho = P.mass * P.wcb * (wf + P.gamma1 * wg);
    float pr = P.k * (rho - P.rho0);
    if (P.clampP) pr = fmaxf(pr, 0.0f);
    s.aux[li] = make_float2(rho, __fdividef(pr, rho * rho));
}

// Forces, wall, kick-drift of own slot j -> rpv[j]; body partial and Verlet displacement in acc.
// Returns a status code (0 ok, 1 non-finite, 2 |x| > 1e9).
__device__ __forceinline__ int res_force(const DevParams& P, const ResParams& R, const ResSmem& s,
                                         const Geom& gm, float damping, int j, BodyAcc& acc) {
    const int li = R.HCAP + j;
    const float4 xi = s.pv[li];
    const float2 ai = s.aux[li];
    float sx = 0.0f, sy = 0.0f;
    const int n = s.ncnt[j];
    if (n != NL_OVERFLOW) {
        const uint2* nq = s.nbr + j;
        uint2 wn = *nq;
        float2 sacc = make_float2(0.0f, 0.0f);
        for (int k = 0; k < n; k += 4) {
            const uint2 w = wn;
            nq += R.S;
            if (k + 4 < n) wn = *nq;
            const int d0 = quad_idx(w, 0), d1 = quad_idx(w, 1);
            pair_force2(P, xi, ai, s.pv[d0], s.aux[d0], s.pv[d1], s.aux[d1], sacc);
            if (k + 2 < n) {
                const int d2 = quad_idx(w, 2), d3 = quad_idx(w, 3);
                pair_force2(P, xi, ai, s.pv[d2], s.aux[d2], s.pv[d3], s.aux[d3], sacc);
            }
        }
        sx = sacc.x;
        sy = sacc.y;
    } else {
        res_cell_candidates(P, R, s, li, [&](int w) { pair_force(P, xi, ai, s.pv[w], s.aux[w], w != li, sx, sy); });
    }
    float gxs = 0.0f, gys = 0.0f, tq = 0.0f;
    const float cp = P.gsign2m2 * ai.y;                    // wall pressure coefficient
    const float cvb = __fdividef(P.m2 * P.beta, ai.x);      // m^2 beta / rho_i
    for_ghost_candidates(P, gm, make_float2(xi.x, xi.y), P.ghost_K1, P.wall1_r2, [&](int g) {
        const float4 xg = s.gst[g];
        float dx = __fsub_rn(xi.x, xg.x), dy = __fsub_rn(xi.y, xg.y);
        if (dist2(dx, dy) < P.h2) {
            const float4 lo = s.glo[g];
            dx -= lo.x;
            dy -= lo.y;
            const float r2 = dx * dx + dy * dy;
            if (!(r2 > 0.0f)) return;
            const float rs = rsqrtf(r2);
            const float hr = P.h - r2 * rs;
            const float gw = P.dws3 * hr * hr * rs;
            const float vr = (xi.z - xg.z) * dx + (xi.w - xg.w) * dy;
            const float cv = __fdividef(cvb * fminf(vr, 0.0f), r2 + P.eps_h2);
            const float c = (cp + cv) * gw;
            const float Gx = c * dx, Gy = c * dy;
            gxs += Gx;
            gys += Gy;
            tq -= lo.z * Gy - lo.w * Gx;     // (r_g - r) x (-G_ig)
        }
    });
    acc.fbx = -gxs;
    acc.fby = -gys;
    acc.tq = tq;
    const float ax = P.mdwcb3 * sx + gxs * P.inv_mass + P.gx;
    const float ay = P.mdwcb3 * sy + gys * P.inv_mass + P.gy;
    float4 xn;
    xn.z = xi.z + P.dt * ax;
    xn.w = xi.w + P.dt * ay;
    xn.x = xi.x + P.dt * xn.z;
    xn.y = xi.y + P.dt * xn.w;
    xn.z *= damping;
    xn.w *= damping;
    s.rpv[j] = xn;
    const float2 xb = s.xb[j];
    const float ddx = (xn.x - xb.x) - (gm.rx - s.m->rbx), ddy = (xn.y - xb.y) - (gm.ry - s.m->rby);
    acc.vmax = ddx * ddx + ddy * ddy;
    const float mag = fabsf(xn.x) + fabsf(xn.y) + fabsf(xn.z) + fabsf(xn.w);
    if (!(mag <= 1e9f)) {
        const bool finite = isfinite(xn.x) && isfinite(xn.y) && isfinite(xn.z) && isfinite(xn.w);
        if (!finite || fabsf(xn.x) > 1e9f || fabsf(xn.y) > 1e9f || fabsf(xn.z) > 1e9f || fabsf(xn.w) > 1e9f)
            return finite ? 2 : 1;
    }
    return 0;
}

// ---------------------------------------------------------------------------------------
// The kernel: grid = B * CS CTAs in clusters of CS (cluster c = rollout c), NT threads each
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(RES_MAXT, 1) k_resident(DevParams P, DevPtrs D, ResParams R, TickArgs T) {
    extern __shared__ __align__(16) unsigned char res_base[];
    const ResSmem s = res_smem(R, res_base);
    ResMisc* m = s.m;
    const int b = blockIdx.x / R.CS, r = cl_rank();
    const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarp = NT >> 5;
    RolloutState* rs = D.rs + b;
    const int frozen = rs->frozen;   // cluster-uniform (written only at the end of a launch)
    if (frozen) {   // a failed rollout keeps reporting its frozen state (as k_tick does)
        if (r == 0 && tid == 0 && T.u_seq) {
            const double* body = D.body + (size_t)b * 6;
            const size_t bk = (size_t)b * T.K + T.k;
            float u2 = T.u_seq[bk * 3 + 2];
            if (T.pd) u2 = (float)(T.Kp * ((double)T.theta_ref[bk] - body[2]) - T.Kd * body[5]);
            for (int c = 0; c < 6; ++c) T.y[bk * 6 + c] = (float)body[c];
            if (T.u_applied) {
                T.u_applied[bk * 3] = T.u_seq[bk * 3];
                T.u_applied[bk * 3 + 1] = T.u_seq[bk * 3 + 1];
                T.u_applied[bk * 3 + 2] = u2;
            }
        }
        return;
    }
    const int sp = rs->sp, ip = rs->ip;
    const long long step0 = rs->step;
    const size_t o = (size_t)b * P.N;
    const int lo = r * R.S, n_own = max(0, min(R.S, P.N - lo)), hi = lo + n_own;
    const int nunit = (n_own + 31) >> 5;
    // ---- tick start: y_k before u_k, ZOH / PD input, state in ----
    if (tid == 0) {
        const double* body = D.body + (size_t)b * 6;
        for (int c = 0; c < 6; ++c) m->body[c] = body[c];
        sincos(m->body[2], &m->body[7], &m->body[6]);
        float u0, u1, u2;
        if (T.u_seq) {
            const size_t bk = (size_t)b * T.K + T.k;
            u0 = T.u_seq[bk * 3];
            u1 = T.u_seq[bk * 3 + 1];
            u2 = T.u_seq[bk * 3 + 2];
            if (T.pd) u2 = (float)(T.Kp * ((double)T.theta_ref[bk] - m->body[2]) - T.Kd * m->body[5]);
            if (r == 0) {
                for (int c = 0; c < 6; ++c) T.y[bk * 6 + c] = (float)m->body[c];
                if (T.u_applied) {
                    T.u_applied[bk * 3] = u0;
                    T.u_applied[bk * 3 + 1] = u1;
                    T.u_applied[bk * 3 + 2] = u2;
                }
                D.u_cur[(size_t)b * 3] = u0;
                D.u_cur[(size_t)b * 3 + 1] = u1;
                D.u_cur[(size_t)b * 3 + 2] = u2;
            }
        } else {
            u0 = D.u_cur[(size_t)b * 3];
            u1 = D.u_cur[(size_t)b * 3 + 1];
            u2 = D.u_cur[(size_t)b * 3 + 2];
        }
        m->u[0] = u0;
        m->u[1] = u1;
        m->u[2] = u2;
        m->need_rebin = 1;
        m->stop = 0;
        m->n_reb = 0;
        m->it_done = 0;
        m->disp = rs->disp;
        m->skin = rs->skin;
        m->rl2 = rs->rl2;
        m->rdisp = rs->rdisp;
        m->last_reb = rs->last_reb;
    }
    if (tid < RES_MAXCS) m->bad_all[tid] = 0;
    // lists of the last rebuild still valid (rs->need_rebin == 0): reload them instead of
    // rebuilding, so the rebuild schedule -- and the bits -- do not depend on how a horizon is
    // split into calls (sph_step(n) twice == sph_step(2n))
    const int reload = !rs->need_rebin;
    for (int j = tid; j < n_own; j += NT) {
        const float4 x = D.pv[sp][o + lo + j];
        const uint32_t k = (D.skey[o + lo + j] << R.IDB) | D.id[ip][o + lo + j];
        s.pv[R.HCAP + j] = x;
        s.key[R.HCAP + j] = k;
        if (reload) {
            s.rpv[j] = x;
            s.rkey[j] = k;
            s.aux[R.HCAP + j] = D.xb[o + lo + j];
        }
    }
    if (reload && tid == 0) {
        m->rbx = rs->rbx;
        m->rby = rs->rby;
        m->need_rebin = 0;
    }
    for (int g = tid; g < P.G; g += NT) s.ghb[g] = __ldg(D.ghost_b + g);
    __syncthreads();
    res_ghosts(P, D, s);
    cl_sync();   // bad_all initialised in every CTA before anyone may write it remotely
    if (reload) res_window<true>(P, R, s, rs, r, lo, n_own, step0);
    const int q0 = lo >> 5;   // global 32-slot group of own unit 0
    for (int it = 0; it < T.n_sub; ++it) {
        const long long step = step0 + it;
        RES_MARK(T, 0, it);
        if (m->need_rebin) res_rebuild(P, R, s, rs, r, lo, n_own, step);
        RES_MARK(T, 1, it);
        const Geom gm = res_geom(m, T.ghost_angle0);
        for (int u = warp; u < nunit; u += nwarp) {
            const int j = u * 32 + lane;
            if (j < n_own) res_density(P, R, s, gm, j);
        }
        RES_MARK(T, 2, it);
        cl_sync();   // A: every CTA's own (rho, P/rho^2) written
        RES_MARK(T, 3, it);
        const int wlo = m->wlo, whi = m->whi, nlow = lo - wlo, nhigh = whi - hi;
        for (int q = tid; q < nlow + nhigh; q += NT) {
            const int g = q < nlow ? wlo + q : hi + (q - nlow);
            const int ow = g / R.S;
            s.aux[R.HCAP + (g - lo)] = cl_map(s.aux, ow)[R.HCAP + g - ow * R.S];
        }
        __syncthreads();
        int bad = 0;
        for (int u = warp; u < nunit; u += nwarp) {
            const int j = u * 32 + lane;
            BodyAcc acc;
            if (j < n_own) {
                const int code = res_force(P, R, s, gm, T.damping, j, acc);
                if (code) {
                    set_status_at(rs, code, (int)(s.key[R.HCAP + j] & R.idmask), step);
                    bad = code;
                }
            }
            // per-warp partial (see write_partial): warp butterfly, one fp64 partial per 32-slot
            // group, stored into every CTA of the cluster
            if (__any_sync(0xffffffffu, acc.fbx != 0.0f || acc.fby != 0.0f || acc.tq != 0.0f)) {
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    acc.fbx += __shfl_xor_sync(0xffffffffu, acc.fbx, d);
                    acc.fby += __shfl_xor_sync(0xffffffffu, acc.fby, d);
                    acc.tq += __shfl_xor_sync(0xffffffffu, acc.tq, d);
                }
            }
            acc.vmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(acc.vmax)));
            if (lane < R.CS)
                cl_map(s.part + q0 + u, lane)[0] = make_double4(acc.fbx, acc.fby, acc.tq, acc.vmax);
        }
        if (bad)
            for (int t = 0; t < R.CS; ++t) cl_map(m->bad_all + r, t)[0] = bad;
        RES_MARK(T, 4, it);
        cl_sync();   // B: every CTA's new own state, partials and flags written
        RES_MARK(T, 5, it);
        if (warp != 0) {   // halo state pull + own copy, overlapping warp 0's body step
            for (int q = tid - 32; q < nlow + nhigh; q += NT - 32) {
                const int g = q < nlow ? wlo + q : hi + (q - nlow);
                const int ow = g / R.S;
                s.pv[R.HCAP + (g - lo)] = cl_map(s.rpv, ow)[g - ow * R.S];
            }
            for (int j = tid - 32; j < n_own; j += NT - 32) s.pv[R.HCAP + j] = s.rpv[j];
        } else {
            // fixed-order fp64 reduction of all npart warp partials (identical in every CTA)
            double4 f = make_double4(0, 0, 0, 0);
            for (int q = lane; q < R.npart; q += 32) {
                const double4 v = s.part[q];
                f.x += v.x;
                f.y += v.y;
                f.z += v.z;
                f.w = fmax(f.w, v.w);
            }
            RES_MARKD(T, 6, it, f.x + f.y + f.z + f.w);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                f.x += __shfl_xor_sync(0xffffffffu, f.x, d);
                f.y += __shfl_xor_sync(0xffffffffu, f.y, d);
                f.z += __shfl_xor_sync(0xffffffffu, f.z, d);
                f.w = fmax(f.w, __shfl_xor_sync(0xffffffffu, f.w, d));
            }
            RES_MARKD(T, 7, it, f.x + f.y + f.z + f.w);
            if (lane == 0) {
                double* bd = m->body;
                if (!T.pin) {
                    const double ax = (f.x + (double)m->u[0]) / P.m_body;
                    const double ay = (f.y + (double)m->u[1]) / P.m_body;
                    const double ath = (f.z + (double)m->u[2]) / P.J_body;
                    bd[3] += P.dtd * ax;
                    bd[4] += P.dtd * ay;
                    bd[5] += P.dtd * ath;
                    bd[0] += P.dtd * bd[3];
                    bd[1] += P.dtd * bd[4];
                    bd[2] += P.dtd * bd[5];
                }
                bool fin = true, big = false;
                for (int c = 0; c < 6; ++c) {
                    fin = fin && isfinite(bd[c]);
                    big = big || fabs(bd[c]) > 1e9;
                }
                int stop = 0;
                for (int t = 0; t < R.CS; ++t) stop |= m->bad_all[t];
                if (!fin || big) {
                    if (r == 0) set_status_at(rs, fin ? 2 : 1, -1, step);
                    stop = 1;
                }
                sincos(bd[2], &bd[7], &bd[6]);
                const double d = sqrt(f.w) + P.dtd * sqrt(bd[3] * bd[3] + bd[4] * bd[4]);
                m->disp = (float)d;
                const int nrb = P.rebin_every ? 1 : ((float)d >= m->rdisp ? 1 : 0);
                m->need_rebin = nrb;
                if (nrb && !P.rebin_every) {   // next substep rebuilds: adapt the skin (B5)
                    const float sk = skin_adapt(P, m->skin, step + 1 - m->last_reb);
                    m->skin = sk;
                    skin_set(P, sk, &m->rl2, &m->rdisp);
                    m->last_reb = step + 1;
                }
                m->it_done = it + 1;
                m->stop = stop;
                RES_MARKD(T, 8, it, bd[2]);
            }
        }
        __syncthreads();
        RES_MARK(T, 9, it);
        if (m->stop) break;
        res_ghosts(P, D, s);
        __syncthreads();
        RES_MARK(T, 10, it);
    }
    // ---- tick end: state out (sorted slots, canonical ids, rebuild-time cells) ----
    for (int j = tid; j < n_own; j += NT) {
        const uint32_t k = s.key[R.HCAP + j];
        D.pv[sp][o + lo + j] = s.pv[R.HCAP + j];
        D.id[ip][o + lo + j] = k & R.idmask;
        D.skey[o + lo + j] = k >> R.IDB;
        D.aux[(size_t)b * P.NA + lo + j] = s.aux[R.HCAP + j];
        D.xb[o + lo + j] = s.xb[j];
    }
    if (r == 0) {
        const double* bd = m->body;
        for (int g = tid; g < P.G; g += NT) {
            const float4 a = s.gst[g], c = s.glo[g];
            D.gst[(size_t)b * P.G + g] = a;
            D.glo[(size_t)b * P.G + g] = make_float2(c.x, c.y);
            D.garm[(size_t)b * P.G + g] = make_float2(c.z, c.w);
        }
        if (tid == 0) {
            double* body = D.body + (size_t)b * 6;
            for (int c = 0; c < 6; ++c) body[c] = bd[c];
            D.geom[b] = res_geom(m, T.ghost_angle0);
            rs->step = step0 + m->it_done;
            rs->rebuilds += m->n_reb;
            rs->need_rebin = m->need_rebin;   // the next launch reloads or rebuilds the lists
            rs->rbx = m->rbx;
            rs->rby = m->rby;
            rs->disp = m->disp;
            rs->skin = m->skin;
            rs->rl2 = m->rl2;
            rs->rdisp = m->rdisp;
            rs->last_reb = m->last_reb;
            if (m->stop) rs->frozen = 1;
        }
    }
    cl_sync();   // no CTA exits while another may still read its shared memory
}

}  // namespace sph
