// sph_kernels.cuh -- the sm_100a kernels of one substep (see sph_device.cuh for the pipeline).
// Included once by sph_api.cu.  P:n = line n of the paper text.
#pragma once
#include <cooperative_groups.h>

#include "sph_device.cuh"

namespace sph {
namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------------------
// Rebuild 1/8: cell key + rank inside the cell (north star: "cell-hash build").
// Grid origin o = float(r_body) - half (reading A19), cells row-major.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void hash_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    RolloutState* rs = D.rs + b;
    if (rs->frozen || !rs->need_rebin) return;
    const int i = bx * TILE + threadIdx.x;
    if (i == 0) {
        rs->span = 0;           // recomputed by k_nlist (kernel boundary orders the atomics)
        rs->rbx = D.geom[b].rx; // body position at this rebuild (Verlet criterion)
        rs->rby = D.geom[b].ry;
    }
    if (i >= P.N) return;
    const size_t o = (size_t)b * P.N;
    const float4 x = D.pv[rs->sp][o + i];
    const Geom gm = D.geom[b];
    const float ox = __fsub_rn(gm.rx, P.half), oy = __fsub_rn(gm.ry, P.half);
    int cx = cell_coord(x.x, ox, P.inv_C), cy = cell_coord(x.y, oy, P.inv_C);
    if (cx < 1 || cx > P.nx - 2 || cy < 1 || cy > P.nx - 2) {   // tunnelled out of the tank
        set_status(rs, 3, (int)D.id[rs->ip][o + i]);
        cx = min(max(cx, 1), P.nx - 2);
        cy = min(max(cy, 1), P.nx - 2);
    }
    const uint32_t c = (uint32_t)(cy * P.nx + cx);
    D.key[o + i] = c;
    D.rank[o + i] = atomicAdd(D.counts + (size_t)b * P.ncell + c, 1u);
}
__global__ void __launch_bounds__(TILE) k_hash(DevParams P, DevPtrs D) { hash_blk(P, D, blockIdx.x, blockIdx.y); }

// ---------------------------------------------------------------------------------------
// Rebuild 2-4/8: segmented exclusive scan of the cell counts of each rollout
//   cstart[b][c] = sum_{c' < c} counts[b][c'],  c = 0..ncell  (cstart[b][ncell] = N).
// Three phases (tile sums, scan of tile sums, down-sweep); the down-sweep re-zeroes counts.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_tot[SCAN_T / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < SCAN_T / 32 ? warp_tot[lane] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
            if (lane >= d) t += y;
        }
        if (lane < SCAN_T / 32) warp_tot[lane] = t;   // inclusive warp prefix
    }
    __syncthreads();
    uint32_t base = w ? warp_tot[w - 1] : 0u;
    if (total) *total = warp_tot[SCAN_T / 32 - 1];
    return base + x - v;
}

__device__ __forceinline__ void scan_reduce_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    if (D.rs[b].frozen || !D.rs[b].need_rebin) return;
    const uint32_t* cnt = D.counts + (size_t)b * P.ncell;
    const int base = bx * SCAN_TILE + threadIdx.x * SCAN_V;
    uint32_t s = 0;
#pragma unroll
    for (int v = 0; v < SCAN_V; ++v) {
        int c = base + v;
        if (c < P.ncell) s += cnt[c];
    }
    uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) D.tsum[(size_t)b * P.nscan + bx] = tot;
}
__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(DevParams P, DevPtrs D) { scan_reduce_blk(P, D, blockIdx.x, blockIdx.y); }

__device__ __forceinline__ void scan_tiles_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = bx;
    if (D.rs[b].frozen || !D.rs[b].need_rebin) return;
    uint32_t* ts = D.tsum + (size_t)b * P.nscan;
    const int per = (P.nscan + SCAN_T - 1) / SCAN_T;   // host guarantees per <= SCAN_V
    uint32_t v[SCAN_V];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k) {
        int t = threadIdx.x * per + k;
        v[k] = (k < per && t < P.nscan) ? ts[t] : 0u;
        s += v[k];
    }
    uint32_t run = block_excl_scan(s, nullptr);
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k) {
        int t = threadIdx.x * per + k;
        if (k < per && t < P.nscan) ts[t] = run;
        run += v[k];
    }
}
__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(DevParams P, DevPtrs D) { scan_tiles_blk(P, D, blockIdx.x, blockIdx.y); }

__device__ __forceinline__ void scan_down_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    if (D.rs[b].frozen || !D.rs[b].need_rebin) return;
    uint32_t* cnt = D.counts + (size_t)b * P.ncell;
    uint32_t* cs = D.cstart + (size_t)b * (P.ncell + 1);
    const int base = bx * SCAN_TILE + threadIdx.x * SCAN_V;
    uint32_t v[SCAN_V];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k) {
        int c = base + k;
        v[k] = c < P.ncell ? cnt[c] : 0u;
        s += v[k];
    }
    uint32_t run = block_excl_scan(s, nullptr) + D.tsum[(size_t)b * P.nscan + bx];
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k) {
        int c = base + k;
        if (c <= P.ncell) cs[c] = run;
        if (c < P.ncell) cnt[c] = 0u;          // counts stay zero between rebuilds
        run += v[k];
    }
}
__global__ void __launch_bounds__(SCAN_T) k_scan_down(DevParams P, DevPtrs D) { scan_down_blk(P, D, blockIdx.x, blockIdx.y); }

// ---------------------------------------------------------------------------------------
// Rebuild 5/8: scatter old slot -> new slot (cell start + rank).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void scatter_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    if (D.rs[b].frozen || !D.rs[b].need_rebin) return;
    const int i = bx * TILE + threadIdx.x;
    if (i >= P.N) return;
    const size_t o = (size_t)b * P.N;
    const uint32_t c = D.key[o + i];
    D.perm[o + D.cstart[(size_t)b * (P.ncell + 1) + c] + D.rank[o + i]] = (uint32_t)i;
}
__global__ void __launch_bounds__(TILE) k_scatter(DevParams P, DevPtrs D) { scatter_blk(P, D, blockIdx.x, blockIdx.y); }

// ---------------------------------------------------------------------------------------
// Rebuild 6/8: make the order inside every cell ascending in canonical id (the atomic ranks
// are not deterministic; this makes the whole sort deterministic and history independent,
// reading A20).  One thread per cell.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void cellsort_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    const RolloutState* rs = D.rs + b;
    if (rs->frozen || !rs->need_rebin) return;
    const int c = bx * TILE + threadIdx.x;
    if (c >= P.ncell) return;
    const uint32_t* cs = D.cstart + (size_t)b * (P.ncell + 1);
    const uint32_t s = cs[c], e = cs[c + 1];
    const int n = (int)(e - s);
    if (n <= 1) return;
    const size_t o = (size_t)b * P.N;
    uint32_t* pm = D.perm + o + s;
    const uint32_t* id = D.id[rs->ip] + o;
    if (n <= SORT_LOCAL) {
        uint32_t src[SORT_LOCAL], key[SORT_LOCAL];
        for (int t = 0; t < n; ++t) {
            src[t] = pm[t];
            key[t] = id[src[t]];
        }
        for (int t = 1; t < n; ++t) {
            uint32_t ks = key[t], ss = src[t];
            int u = t - 1;
            while (u >= 0 && key[u] > ks) {
                key[u + 1] = key[u];
                src[u + 1] = src[u];
                --u;
            }
            key[u + 1] = ks;
            src[u + 1] = ss;
        }
        for (int t = 0; t < n; ++t) pm[t] = src[t];
    } else {   // crowded cell (compressed flow): in-place insertion sort in global memory
        for (int t = 1; t < n; ++t) {
            uint32_t ss = pm[t], ks = id[ss];
            int u = t - 1;
            while (u >= 0 && id[pm[u]] > ks) {
                pm[u + 1] = pm[u];
                --u;
            }
            pm[u + 1] = ss;
        }
    }
}
__global__ void __launch_bounds__(TILE) k_cellsort(DevParams P, DevPtrs D) { cellsort_blk(P, D, blockIdx.x, blockIdx.y); }

// ---------------------------------------------------------------------------------------
// Rebuild 7/8: gather the state into cell order (coalesced writes; reads are nearly sequential
// because particles move little between rebuilds).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void gather_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    const RolloutState* rs = D.rs + b;
    if (rs->frozen || !rs->need_rebin) return;
    const int d = bx * TILE + threadIdx.x;
    if (d >= P.N) return;
    const size_t o = (size_t)b * P.N;
    const int sp = rs->sp, ip = rs->ip;
    const uint32_t src = D.perm[o + d];
    D.pv[sp ^ 1][o + d] = D.pv[sp][o + src];
    D.id[ip ^ 1][o + d] = D.id[ip][o + src];
    D.skey[o + d] = D.key[o + src];
    const float4 x = D.pv[sp ^ 1][o + d];
    D.xb[o + d] = make_float2(x.x, x.y);   // positions at this rebuild (Verlet criterion)
    if (P.perpart) D.hs[o + d] = half_skin(P, x, D.geom[b]);
}
__global__ void __launch_bounds__(TILE) k_gather(DevParams P, DevPtrs D) { gather_blk(P, D, blockIdx.x, blockIdx.y); }

// ---------------------------------------------------------------------------------------
// Rebuild 8/8: neighbour candidate list of every slot: all j != i of the 3x3 rebuild-time
// cell block with |x_i - x_j|^2 < (2h + skin)^2 (float32), stored as int16 slot offsets,
// four per uint2, in a [KQ][N] interleaved layout (one coalesced 8-byte load per four
// candidates).  Unused entries of the last quad are 0.  Lists longer than KMAX, or offsets
// outside int16, mark the particle for the cell-scan fallback.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(TILE) k_nlist(DevParams P, DevPtrs D);
// ---------------------------------------------------------------------------------------
// Density + EOS (Eq. density_update, Eq. EOS, cubic kernel P:268-271):
//   rho_i = m ( sum_{j : r_ij < 2h} W_cb(r_ij)  [self included]  + gamma1 sum_g W_cb(r_ig) )
//   P_i = k (rho_i - rho0);  stores (rho_i, P_i / rho_i^2).
// The list is walked four candidates at a time: one 8-byte offset load, four independent
// 16-byte state loads, then branch-free masked arithmetic.
// ---------------------------------------------------------------------------------------
// W_cb polynomial of a list candidate (no validity mask: list padding points at the particle
// itself and contributes exactly W(0) = 4, which the caller subtracts).  Support by shape, not
// by predicate: W = max(2-q,0)^3 - 4 max(1-q,0)^3 is the cubic spline (Eq. cubicspline) for
// every q >= 0 and exactly 0 beyond 2h; it differs from masking with the canonical predicate
// r2 < (2h)^2 only by O(eps^3) at the rounding boundary (the neighbour SETS stay canonical:
// they are fixed when the lists are built, reading A19).
__device__ __forceinline__ float w_list(const DevParams& P, float4 xi, float4 xj) {
    const float dx = xi.x - xj.x, dy = xi.y - xj.y;
    const float r2 = fmaf(dx, dx, dy * dy);
    const float q = sqrt_approx(r2) * P.inv_h;                  // exactly 0 at r2 = 0
    const float a = fmaxf(2.0f - q, 0.0f), c = fmaxf(1.0f - q, 0.0f);
    return fmaf(-4.0f * c, c * c, a * a * a);
}

#ifndef SPH_F32X2
#define SPH_F32X2 1   // packed FP32 (FADD2 / FMUL2 / FFMA2) list loops
#endif

__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
// c - a as one FFMA2 (a * -1 + c is exact up to the one rounding of the difference; an explicit
// negation of a register operand would cost an FADD per lane under -ftz)
__device__ __forceinline__ float2 rsub2(float2 c, float2 a) { return __ffma2_rn(a, bc2(-1.0f), c); }
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// w_list of two candidates a, b on the packed FP32 pipe (sm_100 FADD2 / FMUL2 / FFMA2): lane
// a / b of every float2 is candidate a / b, with w_list's operations and rounding per lane; one
// issue slot serves both candidates except for the square roots and the clamps.  Returns w_a + w_b.
__device__ __forceinline__ float w_list2(const DevParams& P, float2 pi, float2 xa, float2 xb) {
    const float2 da = rsub2(pi, xa), db = rsub2(pi, xb);
    const float2 r2 = make_float2(fmaf(da.x, da.x, da.y * da.y), fmaf(db.x, db.x, db.y * db.y));
    const float2 q = __fmul2_rn(make_float2(sqrt_approx(r2.x), sqrt_approx(r2.y)), bc2(P.inv_h));
    const float2 a0 = rsub2(bc2(2.0f), q), c0 = rsub2(bc2(1.0f), q);
    const float2 a = make_float2(fmaxf(a0.x, 0.0f), fmaxf(a0.y, 0.0f));
    const float2 c = make_float2(fmaxf(c0.x, 0.0f), fmaxf(c0.y, 0.0f));
    const float2 w = __ffma2_rn(__fmul2_rn(bc2(-4.0f), c), __fmul2_rn(c, c),
                                __fmul2_rn(__fmul2_rn(a, a), a));
    return w.x + w.y;
}

// cell-scan fallback: candidates include the particle itself (valid = false)
__device__ __forceinline__ float w_masked(const DevParams& P, float4 xi, float4 xj, bool valid) {
    const float w = w_list(P, xi, xj);
    return valid ? w : 0.0f;
}

// Load through the read-only path unless the data was written earlier in the same kernel.
template <bool NC, class T>
__device__ __forceinline__ T ld(const T* p) {
    if constexpr (NC) return __ldg(p);
    else return *p;
}

// Wall term gamma1 sum_g W_cb(r_ig) (Eq. density_update), EOS, and the (rho, P/rho^2) store,
// given the fluid sum wf (self term included, in units of C/h^2).
// NC = false: coherent loads (k_coop reads ghost rows that an earlier phase of the same launch
// wrote; the read-only path is only defined for data constant over the whole kernel)
template <bool NC = true>
__device__ __forceinline__ void finish_density(const DevParams& P, const DevPtrs& D, int b, int i,
                                               float2 xi, float wf) {
    float wg = 0.0f;
    const Geom gm = D.geom[b];
    const float4* gst = D.gst + (size_t)b * P.G;
    const float2* glo = D.glo + (size_t)b * P.G;
    for_ghost_candidates(P, gm, xi, P.ghost_K, P.wall_r2, [&](int g) {
        const float4 xg = ld<NC>(gst + g);
        const float dx = __fsub_rn(xi.x, xg.x), dy = __fsub_rn(xi.y, xg.y);
        if (dist2(dx, dy) < P.H2) {
            const float2 lo = ld<NC>(glo + g);
            const float ex = dx - lo.x, ey = dy - lo.y;
            const float r2 = ex * ex + ey * ey;
            wg += wcb_poly(r2 > 0.0f ? r2 * rsqrtf(r2) * P.inv_h : 0.0f);
        }
    });
    const float rho = P.mass * P.wcb * (wf + P.gamma1 * wg);
    float pr = P.k * (rho - P.rho0);
    if (P.clampP) pr = fmaxf(pr, 0.0f);
    D.aux[(size_t)b * P.NA + i] = make_float2(rho, __fdividef(pr, rho * rho));
}

// Density + EOS of slot i of rollout b.  pos(j) returns the (x, y) of list neighbour j of the
// rollout; posg(j) that of a cell-scan candidate (list overflow).
// wn0 / n: the list's first offset quad and length, loaded by the caller.  (Loading them before
// k_density's rollout-state check measured 4 us slower on C3; in k_force it pays, see force_tile.)
template <bool NC, class PosF, class PosG>
__device__ __forceinline__ void density_core(const DevParams& P, const DevPtrs& D, int b, int i,
                                             PosF&& pos, PosG&& posg, uint2 wn0, int n) {
    const size_t o = (size_t)b * P.N;
    const float2 p = pos((uint32_t)i);
    const float4 xi = make_float4(p.x, p.y, 0.f, 0.f);
    float wf = 4.0f;   // self term W_cb(0) ("all particles"): (2-0)^3 - 4 (1-0)^3 = 4
    const uint2* __restrict__ nq = D.nbr + (size_t)b * KQ * P.N + i;
    uint2 wn = wn0;   // the next quad's offsets stay in flight while this one is evaluated
    auto as4 = [](float2 v) { return make_float4(v.x, v.y, 0.f, 0.f); };
    if (n != NL_OVERFLOW) {
        for (int k = 0; k < n; k += 4) {
            const uint2 w = wn;
            nq += P.N;
            if (k + 4 < n) wn = ld<NC>(nq);
#if SPH_F32X2
            wf += w_list2(P, p, pos((uint32_t)(i + quad_offset(w, 0))),
                          pos((uint32_t)(i + quad_offset(w, 1))));
            if (k + 2 < n)     // pairs granularity (see force_list)
                wf += w_list2(P, p, pos((uint32_t)(i + quad_offset(w, 2))),
                              pos((uint32_t)(i + quad_offset(w, 3))));
#else
            const float4 x0 = as4(pos((uint32_t)(i + quad_offset(w, 0))));
            const float4 x1 = as4(pos((uint32_t)(i + quad_offset(w, 1))));
            wf += w_list(P, xi, x0) + w_list(P, xi, x1);
            if (k + 2 < n) {   // pairs granularity (see force_list)
                const float4 x2 = as4(pos((uint32_t)(i + quad_offset(w, 2))));
                const float4 x3 = as4(pos((uint32_t)(i + quad_offset(w, 3))));
                wf += w_list(P, xi, x2) + w_list(P, xi, x3);
            }
#endif
        }
        wf -= 4.0f * (float)(((n + 1) & ~1) - n);   // padding entries (self) added W(0) = 4 each
    } else {
        for_cell_candidates(P, D.cstart + (size_t)b * (P.ncell + 1), ld<NC>(D.skey + o + i),
                            [&](uint32_t j) { wf += w_masked(P, xi, as4(posg(j)), j != (uint32_t)i); });
    }
    finish_density<NC>(P, D, b, i, p, wf);
}

template <bool NC, class PosF, class PosG>
__device__ __forceinline__ void density_core(const DevParams& P, const DevPtrs& D, int b, int i,
                                             PosF&& pos, PosG&& posg) {
    // first offsets, independent of the count load
    const uint2 wn = ld<NC>(D.nbr + (size_t)b * KQ * P.N + i);
    const int n = ld<NC>(D.ncnt + (size_t)b * P.N + i);
    density_core<NC>(P, D, b, i, pos, posg, wn, n);
}

template <bool NC, class PosF>
__device__ __forceinline__ void density_core(const DevParams& P, const DevPtrs& D, int b, int i,
                                             PosF&& pos) {
    density_core<NC>(P, D, b, i, pos, pos);
}

template <bool NC>
__device__ __forceinline__ void density_at(const DevParams& P, const DevPtrs& D, int b, int i,
                                           const float4* __restrict__ pv_) {
    const float4* __restrict__ pv = opaque(pv_);
    density_core<NC>(P, D, b, i, [&](uint32_t j) {
        const float4 v = ld<NC>(pv + j);
        return make_float2(v.x, v.y);
    });
}

// L2 prefetch ahead of the wave: thread 0 of a CTA bulk-prefetches (cp.async.bulk.prefetch.L2)
// the inputs of the tile `dist` CTAs later in launch order (same grid shape) -- the tile a CTA
// starting about one wave later will process -- so its list rows, counts and state come from L2
// instead of DRAM.  Issued after the thread's own work; 1x traffic (each tile once).
template <bool FORCE>
__device__ __forceinline__ void prefetch_ahead(const DevParams& P, const DevPtrs& D, int T, int dist,
                                               bool rev = false) {
    if (threadIdx.x != 0 || dist <= 0) return;
    const long long c = (long long)blockIdx.y * gridDim.x + blockIdx.x + dist;
    if (c >= (long long)gridDim.x * gridDim.y) return;
    const int by = (int)(c / gridDim.x);
    const int b = rev ? (int)gridDim.y - 1 - by : by, t0 = P.own_lo + (int)(c % gridDim.x) * T;
    const int cnt = min(T, P.N - t0);
    if (cnt <= 0) return;
    const size_t o = (size_t)b * P.N;
    auto pf = [](const void* p, size_t bytes) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p);
        const uintptr_t lo = a & ~(uintptr_t)15, hi = (a + bytes + 15) & ~(uintptr_t)15;
        bulk_prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
    };
    for (int q = 0; q < 3; ++q)   // lists of up to 12 entries (p90 of C2: 11)
        pf(D.nbr + (size_t)b * KQ * P.N + (size_t)q * P.N + t0, (size_t)cnt * 8);
    pf(D.ncnt + o + t0, (size_t)cnt);
    const RolloutState* rs = D.rs + b;
    pf(D.pv[rs->sp ^ rs->need_rebin] + o + t0, (size_t)cnt * 16);
    if (FORCE) {
        pf(D.aux + (size_t)b * P.NA + t0, (size_t)cnt * 8);
        pf(D.xb + o + t0, (size_t)cnt * 8);
    }
}

// skip_rebuilding = 1 when rollouts that rebuild this substep get their densities from
// k_nlist_density (which runs concurrently on another branch of the graph).
// Plain variant: neighbour positions gathered from global memory through L1.
// TD slots per CTA: a CTA gathers from [t0 - span, t0 + TD + span), so larger CTAs touch fewer
// window lines per own slot (fewer compulsory L1 misses); TD is chosen on the host.
template <int TD>
__global__ void __launch_bounds__(TD) k_density(DevParams P, DevPtrs D, int skip_rebuilding) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const RolloutState* rs = D.rs + b;
    if (rs->frozen || (skip_rebuilding && rs->need_rebin)) return;   // CTA-uniform
    const int i = P.own_lo + blockIdx.x * TD + threadIdx.x;
    const float4* pv = D.pv[rs->sp ^ rs->need_rebin] + (size_t)b * P.N;
    if (i < P.N) density_at<true>(P, D, b, i, pv);
    prefetch_ahead<false>(P, D, TD, P.pf_d);
}

// ---------------------------------------------------------------------------------------
// Small-rollout rebuild path (N and the cell grid fit in shared memory, e.g. C1, C2, C3):
//   k_rebuild_plan   one CTA compacts the rollouts that need a rebuild into a work list;
//   k_rebuild_small  persistent CTAs, ONE CTA PER LISTED ROLLOUT: counting sort by cell with
//                    shared-memory atomics, block scan, per-cell canonical-id order, gather,
//                    neighbour lists and the densities of the rollout -- all in shared memory,
//                    no grid-wide phases.  It runs concurrently with k_density for the other
//                    rollouts, so a rebuild costs one SM for tens of microseconds instead of
//                    eight grid-wide launches.
// ---------------------------------------------------------------------------------------
constexpr int RB_T = 1024;
constexpr int RBS_T = 1024;   // threads of the per-rollout sort CTA (k_rebuild_small; 512: slower)

template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_t(uint32_t v, uint32_t* total,
                                                      uint32_t* warp_tot /* [NT/32] smem */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < NT / 32 ? warp_tot[lane] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
            if (lane >= d) t += y;
        }
        if (lane < NT / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    const uint32_t base = w ? warp_tot[w - 1] : 0u;
    if (total) *total = warp_tot[NT / 32 - 1];
    __syncthreads();   // warp_tot may be reused by the caller's next scan
    return base + x - v;
}

// set_cond != 0 (graph launch): also sets the IF node that guards the grid-wide rebuild
// kernels, so substeps without any rebuild skip them entirely.
__global__ void __launch_bounds__(RB_T) k_rebuild_plan(DevParams P, DevPtrs D,
                                                       cudaGraphConditionalHandle cond,
                                                       int set_cond) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t wt[RB_T / 32];
    uint32_t base = 0;
    for (int b0 = 0; b0 < P.B; b0 += RB_T) {
        const int b = b0 + threadIdx.x;
        const uint32_t f = (b < P.B && D.rs[b].need_rebin && !D.rs[b].frozen) ? 1u : 0u;
        uint32_t tot;
        const uint32_t pos = base + block_excl_scan_t<RB_T>(f, &tot, wt);
        if (f) D.rlist[pos] = b;
        base += tot;
    }
    if (threadIdx.x == 0) {
        *D.rcount = (int)base;
        if (set_cond) cudaGraphSetConditional(cond, base > 0 ? 1u : 0u);
    }
}

// neighbour candidate list of slot i (see k_nlist) from a given cell-start table
// Returns max |j - i| over the list entries (the staging window of k_density / k_force).
// DENS = true also accumulates the fluid density sum of the appended (2h + skin) candidates
// that lie within 2h into *wf (self term included); on list overflow *wf is not valid.
// PP = false: the per-particle half-skin radius (B6) compiled out (callers check P.perpart).
template <bool DENS = false, bool PP = true, class PosF>
__device__ __forceinline__ int build_list_core(const DevParams& P, const DevPtrs& D, int b, int i,
                                               const uint32_t* cs, uint32_t cell, PosF&& pos,
                                               float* wf_out = nullptr) {
    const size_t o = (size_t)b * P.N;
    const float2 xi = pos((uint32_t)i);
    uint2* nq = D.nbr + (size_t)b * KQ * P.N + i;
    int n = 0, first = 0, last = 0;
    bool ovf = false;
    uint64_t acc = 0;           // the last four offsets, oldest in the low 16 bits
    float wf = 4.0f;            // self term W_cb(0)
    // SIMT-friendly: a branch-free hit mask over up to 32 candidates of a cell-row segment
    // (shift-in, bit 0 = last candidate), then only the set bits are appended, highest bit
    // first (= ascending j, the order of a plain scan).
    const int cy = (int)cell / P.nx, cx = (int)cell - cy * P.nx;
    const float RL2u = D.rs[b].rl2;  // this rollout's list radius^2 (uniform / B5 skin)
    const float* __restrict__ hs = D.hs + o;
    const float hsi = PP && P.perpart ? hs[i] : 0.0f;
    for (int dy = -1; dy <= 1 && !ovf; ++dy) {
        const int c0 = (cy + dy) * P.nx + cx - 1;
        const int j0 = (int)cs[c0], j1 = (int)cs[c0 + 3];
        for (int base = j0; base < j1 && !ovf; base += 32) {
            const int cnt = min(32, j1 - base);
            uint32_t m = 0u;
            for (int k = 0; k < cnt; ++k) {
                const float2 xj = pos((uint32_t)(base + k));
#if SPH_F32X2
                // the canonical predicate on the packed pipe: (x_i - x_j, y_i - y_j) in one FFMA2
                // (x_j * -1 + x_i: one rounding, = __fsub_rn), squares in one FMUL2, then the
                // same __fadd_rn -- bit-identical to dist2(__fsub_rn(..), __fsub_rn(..))
                const float2 dd = rsub2(xi, xj);
                const float2 sq = __fmul2_rn(dd, dd);
                const float r2 = __fadd_rn(sq.x, sq.y);
#else
                const float r2 = dist2(__fsub_rn(xi.x, xj.x), __fsub_rn(xi.y, xj.y));
#endif
                // list radius: 2h + skin, or 2h + hs_i + hs_j (per-particle skins, B6)
                float RL2 = RL2u;
                if (PP && P.perpart) {
                    const float RL = __fadd_rn(P.Hf, __fadd_rn(hsi, hs[base + k]));
                    RL2 = __fmul_rn(RL, RL);
                }
                m = (m << 1) | (r2 < RL2 ? 1u : 0u);
            }
            const int self = i - base;
            if (self >= 0 && self < cnt) m &= ~(1u << (cnt - 1 - self));
            while (m != 0u) {
                const int p = 31 - __clz(m);
                m ^= 1u << p;
                const int j = base + cnt - 1 - p;
                const int off = j - i;
                if (n >= KMAX || (unsigned)(off + 32768) > 65535u) {
                    ovf = true;
                    break;
                }
                first = n == 0 ? off : first;
                last = off;
                acc = (acc >> 16) | ((uint64_t)(uint16_t)(int16_t)off << 48);
                if ((++n & 3) == 0) {
                    *nq = make_uint2((uint32_t)acc, (uint32_t)(acc >> 32));
                    nq += P.N;
                }
                if (DENS) {
                    const float2 xj = pos((uint32_t)j);
                    wf += w_list(P, make_float4(xi.x, xi.y, 0.f, 0.f), make_float4(xj.x, xj.y, 0.f, 0.f));
                }
            }
        }
    }
    if (!ovf && (n & 3)) {   // last partial quad: align to the low lanes, pad with 0 (= self)
        acc >>= 16 * (4 - (n & 3));
        *nq = make_uint2((uint32_t)acc, (uint32_t)(acc >> 32));
    }
    D.ncnt[o + i] = (uint8_t)(ovf ? NL_OVERFLOW : n);
    if (DENS && wf_out) *wf_out = wf;
    return ovf ? -1 : max(-first, last);   // entries ascend in j: first = min, last = max
}

__device__ __forceinline__ void nlist_blk(const DevParams& P, const DevPtrs& D, int bx, int by) {
    const int b = by;
    RolloutState* rs = D.rs + b;
    if (rs->frozen || !rs->need_rebin) return;
    const int i = bx * TILE + threadIdx.x;
    int span = 0;
    if (i < P.N) {
        const size_t o = (size_t)b * P.N;
        const float4* pv = D.pv[rs->sp ^ 1] + o;
        span = build_list_core(P, D, b, i, D.cstart + (size_t)b * (P.ncell + 1), D.skey[o + i],
                               [&](uint32_t j) {
                                   const float4 v = __ldg(pv + j);
                                   return make_float2(v.x, v.y);
                               });
    }
    span = __reduce_max_sync(0xffffffffu, span);
    if ((threadIdx.x & 31) == 0 && span > 0) atomicMax(&rs->span, span);
}
__global__ void __launch_bounds__(TILE) k_nlist(DevParams P, DevPtrs D) { nlist_blk(P, D, blockIdx.x, blockIdx.y); }

// dynamic shared memory: start[ncell + 1] u32 | key[N] u32 | perm[N] u32 | id[N] u32 | rank[N] u16
// (host guarantees N < 65536).  Sort only: the lists and the densities of the rebuilt rollouts
// follow grid-wide in k_nlist_density.
__global__ void __launch_bounds__(RBS_T) k_rebuild_small(DevParams P, DevPtrs D) {
    extern __shared__ uint32_t smem[];
    __shared__ uint32_t wt[RBS_T / 32];
    uint32_t* s_start = smem;
    uint32_t* s_key = s_start + ((P.ncell + 1 + 3) & ~3);   // 16-byte aligned (float2 alias)
    uint32_t* s_perm = s_key + P.N;
    uint32_t* s_id = s_perm + P.N;   // canonical ids of the unsorted slots (step 4's keys)
    uint16_t* s_rank = reinterpret_cast<uint16_t*>(s_id + P.N);
    const int count = *D.rcount;
    const int T = RBS_T, tid = threadIdx.x;
    // active CTAs: about one per 3.5 rebuilding rollouts, at least gridDim / 8 -- every resident
    // 1024-thread sort CTA takes half an SM from the concurrent densities / forces, so a few CTAs
    // each sorting several rollouts beat one per rollout (C3 window 97.3 -> 96.6 ms per tick at
    // 18 CTAs, but 9.3 G/s at the horizon's steady state; 74 CTAs: 13.0 -> 13.3 G/s there).
    // Which CTA sorts a rollout does not change its bits.
    const int G = min((int)gridDim.x, max((int)gridDim.x / 8, (2 * count + 6) / 7));
    if ((int)blockIdx.x >= G) return;
    for (int w = blockIdx.x; w < count; w += G) {
        const int b = D.rlist[w];
        RolloutState* rs = D.rs + b;
        const int sp = rs->sp, ip = rs->ip;
        const size_t o = (size_t)b * P.N;
        const float4* pv0 = D.pv[sp] + o;
        float4* pv1 = D.pv[sp ^ 1] + o;
        const uint32_t* id0 = D.id[ip] + o;
        uint32_t* id1 = D.id[ip ^ 1] + o;
        for (int c = tid; c <= P.ncell; c += T) s_start[c] = 0u;
        __syncthreads();
        // 1. cell key + rank (shared-memory atomics)
        const Geom gm = D.geom[b];
        const float ox = __fsub_rn(gm.rx, P.half), oy = __fsub_rn(gm.ry, P.half);
        for (int i = tid; i < P.N; i += T) {
            const float4 x = pv0[i];
            int cx = cell_coord(x.x, ox, P.inv_C), cy = cell_coord(x.y, oy, P.inv_C);
            if (cx < 1 || cx > P.nx - 2 || cy < 1 || cy > P.nx - 2) {
                set_status(rs, 3, (int)id0[i]);
                cx = min(max(cx, 1), P.nx - 2);
                cy = min(max(cy, 1), P.nx - 2);
            }
            const uint32_t c = (uint32_t)(cy * P.nx + cx);
            s_key[i] = c;
            s_id[i] = id0[i];
            s_rank[i] = (uint16_t)atomicAdd(s_start + c, 1u);
        }
        __syncthreads();
        // 2. exclusive scan of the counts -> cell starts (smem and global table)
        {
            const int per = (P.ncell + 1 + T - 1) / T;
            const int c0 = tid * per;
            uint32_t s = 0;
            for (int k = 0; k < per; ++k)
                if (c0 + k <= P.ncell) s += s_start[c0 + k];
            uint32_t run = block_excl_scan_t<RBS_T>(s, nullptr, wt);
            uint32_t* cs = D.cstart + (size_t)b * (P.ncell + 1);
            for (int k = 0; k < per; ++k) {
                const int c = c0 + k;
                if (c <= P.ncell) {
                    const uint32_t v = s_start[c];
                    s_start[c] = run;
                    cs[c] = run;
                    run += v;
                }
            }
        }
        __syncthreads();
        // 3. scatter
        for (int i = tid; i < P.N; i += T) s_perm[s_start[s_key[i]] + s_rank[i]] = (uint32_t)i;
        __syncthreads();
        // 4. canonical-id order inside each cell (reading A20)
        for (int c = tid; c < P.ncell; c += T) {
            const int s = (int)s_start[c], e = (int)s_start[c + 1];
            for (int t = s + 1; t < e; ++t) {
                const uint32_t ss = s_perm[t], ks = s_id[ss];
                int u = t - 1;
                while (u >= s && s_id[s_perm[u]] > ks) {
                    s_perm[u + 1] = s_perm[u];
                    --u;
                }
                s_perm[u + 1] = ss;
            }
        }
        __syncthreads();
        // 5. gather into cell order
        for (int d = tid; d < P.N; d += T) {
            const uint32_t src = s_perm[d];
            const float4 v = pv0[src];
            pv1[d] = v;
            id1[d] = s_id[src];
            const uint32_t c = s_key[src];
            D.skey[o + d] = c;
            D.xb[o + d] = make_float2(v.x, v.y);   // positions at this rebuild (Verlet)
            if (P.perpart) D.hs[o + d] = half_skin(P, v, gm);
        }
        __syncthreads();
        // lists + densities follow in k_nlist_density (grid-wide)
        if (tid == 0) {
            rs->span = 0;
            rs->rbx = gm.rx;     // body position at this rebuild (Verlet criterion)
            rs->rby = gm.ry;
        }
        __syncthreads();
    }
}

// Neighbour lists + densities of the rollouts in the rebuild work list, grid-wide:
// grid = (tiles, Y); CTA (x, y) handles tile x of work items y, y + Y, ...  The cell table,
// slot cells and sorted state come from the sort (k_rebuild_small or the grid-wide
// rebuild kernels); the list just written by a thread is read back by the same thread.
// lists + density of slot i of the rebuilt rollout b (every lane of the warp calls it)
template <bool NC = true, bool PP = true>
__device__ __forceinline__ void nlist_density_at(const DevParams& P, const DevPtrs& D, int b, int i) {
    RolloutState* rs = D.rs + b;
    const size_t o = (size_t)b * P.N;
    const float4* __restrict__ pv = opaque(D.pv[rs->sp ^ 1] + o);   // sorted (rebuilt) buffer
    auto pos = [&](uint32_t j) {   // (x, y) half of the state: one 8-byte load
        return ld<NC>(reinterpret_cast<const float2*>(pv + j));
    };
    int span = 0;
    if (i < P.N) {
        float wf;
        span = build_list_core<true, PP>(P, D, b, i, D.cstart + (size_t)b * (P.ncell + 1),
                                         D.skey[o + i], pos, &wf);
        if (span >= 0) finish_density<NC>(P, D, b, i, pos((uint32_t)i), wf);
        else density_core<false>(P, D, b, i, pos);   // list overflow: cell-scan density
    }
    span = __reduce_max_sync(0xffffffffu, span);
    if ((threadIdx.x & 31) == 0 && span > 0) atomicMax(&rs->span, span);
}

template <int TN, bool PP>
__global__ void __launch_bounds__(TN) k_nlist_density(DevParams P, DevPtrs D) {
    pdl_wait();
    pdl_trigger();
    const int count = *D.rcount;
    const int i = P.own_lo + blockIdx.x * TN + threadIdx.x;
    for (int w = blockIdx.y; w < count; w += gridDim.y) nlist_density_at<true, PP>(P, D, D.rlist[w], i);
}

// ---------------------------------------------------------------------------------------
// Forces + wall + fluid integration + body partials.
//   F^p_i = m sum m (P_i/rho_i^2 + P_j/rho_j^2) grad W_ij            (Eq. momentum)
//   F^v_i = m sum m 2 alpha h/(rho_i+rho_j) (v_ij.r_ij)/(r^2 + eps h^2) grad W_ij
//   G_ig  = s 2 m^2 (P_i/rho_i^2) grad W_s3 + m^2 beta/rho_i min(v.r,0)/(r^2+eps h^2) grad W_s3
//           (Eqs. pressure_b2f, viscous_b2f P:188-200; s = ghost_pressure_sign, reading A4)
//   a_i = (-F^p + F^v + sum_g G_ig) / m + g        (Algorithm 1 l.8)
//   v_i += dt a_i ; x_i += dt v_i                   (symplectic Euler, kick then drift)
// The reaction -G_ig on the body (Eqs. pressure_f2b, viscous_f2b) and its torque about r are
// reduced per CTA (warp shuffle -> fp64 per warp -> fixed order) into D.part.
// ---------------------------------------------------------------------------------------
// (-pressure + viscous) pair term per m^2, times r_ij, accumulated into (sx, sy).
// The sums (sx, sy) are in units of 3C/h^3: dW/dr = (3C/h^3) d(q) with
// d(q) = q (3q - 4) for q < 1 and -(2 - q)^2 for 1 <= q < 2 (Eq. cubicspline differentiated).
// r2 is clamped before rsqrt, so the self pair and list padding (dx = dy = 0) and coincident
// particles contribute exactly zero (zero gradient at r = 0, reading A8) without a mask.
// d(q) by shape, branch-free: d = 4 max(1-q,0)^2 - max(2-q,0)^2 equals q(3q-4) for q < 1 and
// -(2-q)^2 for 1 <= q < 2, and is exactly 0 beyond 2h (skin candidates of the list); see w_list
// for why no canonical predicate is needed here.
__device__ __forceinline__ void pair_force(const DevParams& P, float4 xi, float2 ai, float4 xj,
                                           float2 aj, float& sx, float& sy) {
    const float dx = xi.x - xj.x, dy = xi.y - xj.y;
    const float r2 = fmaf(dx, dx, dy * dy);
    const float rs = rsqrtf(fmaxf(r2, 1e-30f));                    // 1 / r
    const float q = r2 * rs * P.inv_h;
    const float t = fmaxf(2.0f - q, 0.0f), u = fmaxf(1.0f - q, 0.0f);
    const float d = fmaf(4.0f * u, u, -(t * t));
    const float vr = (xi.z - xj.z) * dx + (xi.w - xj.w) * dy;
    const float visc = __fdividef(P.alpha2h * vr, (ai.x + aj.x) * (r2 + P.eps_h2));
    const float s = (visc - (ai.y + aj.y)) * (d * rs);
    sx += s * dx;
    sy += s * dy;
}

// pair_force of two list pairs a, b on the packed FP32 pipe (see w_list2): lane a / b of every
// float2 is pair a / b with pair_force's operations per lane; the accumulation s = (sx, sy) is
// one FFMA2 per pair, in the order a then b as in two pair_force calls.
__device__ __forceinline__ void pair_force2(const DevParams& P, float4 xi, float2 ai, float4 xa,
                                            float2 aa, float4 xb, float2 ab, float2& s) {
    const float2 pi = make_float2(xi.x, xi.y), vi = make_float2(xi.z, xi.w);
    const float2 da = rsub2(pi, make_float2(xa.x, xa.y)), db = rsub2(pi, make_float2(xb.x, xb.y));
    const float2 wa = rsub2(vi, make_float2(xa.z, xa.w)), wb = rsub2(vi, make_float2(xb.z, xb.w));
    const float2 r2 = make_float2(fmaf(da.x, da.x, da.y * da.y), fmaf(db.x, db.x, db.y * db.y));
    const float2 vr = make_float2(fmaf(wa.x, da.x, wa.y * da.y), fmaf(wb.x, db.x, wb.y * db.y));
    const float2 rs = make_float2(rsqrtf(fmaxf(r2.x, 1e-30f)), rsqrtf(fmaxf(r2.y, 1e-30f)));
    const float2 q = __fmul2_rn(__fmul2_rn(r2, rs), bc2(P.inv_h));
    const float2 t0 = rsub2(bc2(2.0f), q), u0 = rsub2(bc2(1.0f), q);
    const float2 t = make_float2(fmaxf(t0.x, 0.0f), fmaxf(t0.y, 0.0f));
    const float2 u = make_float2(fmaxf(u0.x, 0.0f), fmaxf(u0.y, 0.0f));
    // -d = t^2 - 4u^2 and -(visc - (P_i/rho_i^2 + P_j/rho_j^2)): both factors of the pair
    // scalar negated (exact), so no negated register operand is needed
    const float2 nd = __ffma2_rn(__fmul2_rn(bc2(-4.0f), u), u, __fmul2_rn(t, t));
    const float2 rho = make_float2(ai.x + aa.x, ai.x + ab.x);
    const float2 pp = make_float2(ai.y + aa.y, ai.y + ab.y);
    const float2 den = __fmul2_rn(rho, __fadd2_rn(r2, bc2(P.eps_h2)));
    const float2 nvisc = __fmul2_rn(__fmul2_rn(bc2(-P.alpha2h), vr),
                                    make_float2(rcp_approx(den.x), rcp_approx(den.y)));
    const float2 sc = __fmul2_rn(__fadd2_rn(nvisc, pp), __fmul2_rn(nd, rs));
    s = __ffma2_rn(bc2(sc.x), da, s);
    s = __ffma2_rn(bc2(sc.y), db, s);
}

// masked variant for the cell-scan fallback (candidates may include j == i)
__device__ __forceinline__ void pair_force(const DevParams& P, float4 xi, float2 ai, float4 xj,
                                           float2 aj, bool valid, float& sx, float& sy) {
    float tx = 0.0f, ty = 0.0f;
    pair_force(P, xi, ai, xj, aj, tx, ty);
    if (valid) {
        sx += tx;
        sy += ty;
    }
}

// List walk of the force kernel: four candidates per 8-byte offset load.  PV / AX return the
// state / aux of a neighbour given its signed slot offset from i (pointer arithmetic relative
// to slot i's own address: one PRMT/SHF + one LEA pair per neighbour, no 64-bit index math).
template <bool NC = true, class PV, class AX>
__device__ __forceinline__ void force_list(const DevParams& P, const uint2* __restrict__ nq, int n,
                                           uint2 q0, float4 xi, float2 ai, PV&& pvj, AX&& axj,
                                           float& sx, float& sy) {
    uint2 wn = q0;   // offsets stream from DRAM: keep the next quad's load in flight
#if SPH_F32X2
    float2 s = make_float2(sx, sy);
#endif
    for (int k = 0; k < n; k += 4) {
        const uint2 w = wn;
        nq += P.N;
        if (k + 4 < n) wn = ld<NC>(nq);
        // pairs granularity: the second half of a quad only when some lane of the warp needs it
        // (padding entries are the particle itself: exact zero contribution)
        const int d0 = quad_offset(w, 0), d1 = quad_offset(w, 1);
        const float4 x0 = pvj(d0), x1 = pvj(d1);
        const float2 a0 = axj(d0), a1 = axj(d1);
#if SPH_F32X2
        pair_force2(P, xi, ai, x0, a0, x1, a1, s);
#else
        pair_force(P, xi, ai, x0, a0, sx, sy);
        pair_force(P, xi, ai, x1, a1, sx, sy);
#endif
        if (k + 2 < n) {
            const int d2 = quad_offset(w, 2), d3 = quad_offset(w, 3);
            const float4 x2 = pvj(d2), x3 = pvj(d3);
            const float2 a2 = axj(d2), a3 = axj(d3);
#if SPH_F32X2
            pair_force2(P, xi, ai, x2, a2, x3, a3, s);
#else
            pair_force(P, xi, ai, x2, a2, sx, sy);
            pair_force(P, xi, ai, x3, a3, sx, sy);
#endif
        }
    }
#if SPH_F32X2
    sx = s.x;
    sy = s.y;
#endif
}

#ifndef SPH_FORCE_MINB
#define SPH_FORCE_MINB 5   // 48 registers with the packed pair math (sweep 4..6: 5 best, no loop spill)
#endif

// Body partial accumulators of one thread (reaction force, torque, squared displacement).
struct BodyAcc {
    float fbx = 0.0f, fby = 0.0f, tq = 0.0f, vmax = 0.0f;
};

// Forces, wall, integration and Verlet displacement of slot i (i < N) of rollout b.
// pvj(d) / axj(d) read list neighbour i + d; pv / aux are the rollout's global
// rows (cell-scan fallback of overflowing lists).  The body geometry is loaded after the list
// walk so it does not occupy registers during it.
template <bool NC = true, bool PP = true, class PV, class AX>
__device__ __forceinline__ void force_particle(const DevParams& P, const DevPtrs& D, float damping,
                                               int b, int i, int cur, const RolloutState* rs,
                                               float4 xi, float2 ai,
                                               const float4* __restrict__ pv,
                                               const float2* __restrict__ aux, PV&& pvj, AX&& axj,
                                               BodyAcc& acc, uint2 q0, int n) {
    // q0 / n: the list's first offset quad and length (loaded by the caller, see force_tile)
    const size_t o = (size_t)b * P.N;
    float sx = 0.0f, sy = 0.0f;   // sum of (-pressure + viscous) * grad W / m^2
    const uint2* __restrict__ nq = D.nbr + (size_t)b * KQ * P.N + i;

    if (n != NL_OVERFLOW) {
        force_list<NC>(P, nq, n, q0, xi, ai, pvj, axj, sx, sy);
    } else {
        for_cell_candidates(P, D.cstart + (size_t)b * (P.ncell + 1), D.skey[o + i], [&](uint32_t j) {
            pair_force(P, xi, ai, ld<NC>(pv + j), ld<NC>(aux + j), j != (uint32_t)i, sx, sy);
        });
    }
    const Geom gm = D.geom[b];
    float gxs = 0.0f, gys = 0.0f;   // sum_g G_ig
    const float4* gst = D.gst + (size_t)b * P.G;
    const float2* glo = D.glo + (size_t)b * P.G;
    const float2* garm = D.garm + (size_t)b * P.G;
    const float cp = P.gsign2m2 * ai.y;                    // wall pressure coefficient
    const float cvb = __fdividef(P.m2 * P.beta, ai.x);      // m^2 beta / rho_i
    float tq = 0.0f;
    for_ghost_candidates(P, gm, make_float2(xi.x, xi.y), P.ghost_K1, P.wall1_r2, [&](int g) {
        const float4 xg = ld<NC>(gst + g);
        float dx = __fsub_rn(xi.x, xg.x), dy = __fsub_rn(xi.y, xg.y);
        if (dist2(dx, dy) < P.h2) {
            const float2 lo = ld<NC>(glo + g);
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
            const float2 a = ld<NC>(garm + g);
            tq -= a.x * Gy - a.y * Gx;     // (r_g - r) x (-G_ig)
        }
    });
    acc.fbx = -gxs;
    acc.fby = -gys;
    acc.tq = tq;
    const float ax = P.mdwcb3 * sx + gxs * P.inv_mass + P.gx;   // m * 3C/h^3 * sum
    const float ay = P.mdwcb3 * sy + gys * P.inv_mass + P.gy;
    float4 xn;
    xn.z = xi.z + P.dt * ax;
    xn.w = xi.w + P.dt * ay;
    xn.x = xi.x + P.dt * xn.z;
    xn.y = xi.y + P.dt * xn.w;
    xn.z *= damping;
    xn.w *= damping;
    D.pv[cur ^ 1][o + i] = xn;
    // Verlet criterion on actual displacements: displacement since the last rebuild
    // relative to the body translation since then (k_body adds this step's body drift).
    // vmax carries the squared displacement through the reductions.
    const float2 xb = ld<NC>(D.xb + o + i);
    const float ddx = (xn.x - xb.x) - (gm.rx - rs->rbx), ddy = (xn.y - xb.y) - (gm.ry - rs->rby);
    acc.vmax = ddx * ddx + ddy * ddy;
    if (PP && P.perpart) {   // (|d_i| / hs_i)^2 (B6; PP = false: compiled out of the C3 kernel)
        const float ih = __frcp_rn(ld<NC>(D.hs + o + i));
        acc.vmax *= ih * ih;
    }
    // one test for the common case: the abs-sum is NaN / inf for any non-finite element and
    // exceeds 1e9 whenever an element does; classify only in the rare branch
    const float mag = fabsf(xn.x) + fabsf(xn.y) + fabsf(xn.z) + fabsf(xn.w);
    if (!(mag <= 1e9f)) {
        const bool finite = isfinite(xn.x) && isfinite(xn.y) && isfinite(xn.z) && isfinite(xn.w);
        if (!finite || fabsf(xn.x) > 1e9f || fabsf(xn.y) > 1e9f || fabsf(xn.z) > 1e9f ||
            fabsf(xn.w) > 1e9f)
            set_status(const_cast<RolloutState*>(rs), finite ? 2 : 1,
                       (int)D.id[rs->ip ^ rs->need_rebin][o + i]);
    }
}

// Body partials: warp butterfly (deterministic order), one fp64 partial per warp of 32 slots,
// index q = slot / 32 within the rollout (written straight to global memory, no CTA barrier).
// The wall reaction and torque are zero for warps away from the wall (most of them): their
// butterflies are skipped (the warp-uniform test is exact: a sum of zeros is zero).  The squared
// displacement is >= 0, so its maximum is an unsigned maximum of the bit patterns (one REDUX).
__device__ __forceinline__ void write_partial(const DevParams& P, const DevPtrs& D, int b, int q,
                                              BodyAcc a) {
    if (__any_sync(0xffffffffu, a.fbx != 0.0f || a.fby != 0.0f || a.tq != 0.0f)) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a.fbx += __shfl_xor_sync(0xffffffffu, a.fbx, d);
            a.fby += __shfl_xor_sync(0xffffffffu, a.fby, d);
            a.tq += __shfl_xor_sync(0xffffffffu, a.tq, d);
        }
    }
    a.vmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(a.vmax)));
    if ((threadIdx.x & 31) == 0 && q < P.npart)
        D.part[(size_t)b * P.npart + q] = make_double4(a.fbx, a.fby, a.tq, a.vmax);
}

// List head (first offset quad, length) of slot i of rollout b: independent of the rollout
// state, so the callers issue it before reading that state.
template <bool NC = true>
__device__ __forceinline__ void list_head(const DevParams& P, const DevPtrs& D, int b, int i,
                                          uint2& q0, int& n) {
    q0 = make_uint2(0u, 0u);
    n = 0;
    if (i < P.N) {
        q0 = ld<NC>(D.nbr + (size_t)b * KQ * P.N + i);
        n = D.ncnt[(size_t)b * P.N + i];
    }
}

template <int TF, bool NC = true, bool PP = true>
__device__ __forceinline__ void force_tile(const DevParams& P, const DevPtrs& D, float damping,
                                           int b, int tile) {
    const int i = tile * TF + threadIdx.x;
    uint2 q0;
    int n;
    list_head<NC>(P, D, b, i, q0, n);   // (discarded if the rollout is frozen)
    const RolloutState* rs = D.rs + b;
    if (rs->frozen) return;   // CTA-uniform (before any warp-level collective)
    const int cur = rs->sp ^ rs->need_rebin;
    const float4* __restrict__ pv = D.pv[cur] + (size_t)b * P.N;
    const float2* __restrict__ aux = D.aux + (size_t)b * P.NA;
    BodyAcc acc;
    if (i < P.N) {
        const float4* __restrict__ pvi = opaque(pv + i);
        const float2* __restrict__ axi = opaque(aux + i);
        force_particle<NC, PP>(P, D, damping, b, i, cur, rs, *pvi, *axi, pv, aux,
                           [&](int d) { return ld<NC>(pvi + d); },
                           [&](int d) { return ld<NC>(axi + d); }, acc, q0, n);
    }
    write_partial(P, D, b, i >> 5, acc);
}

// mode 0: every rollout (grid.y = B); 1: rollouts that do NOT rebuild this substep (their
// densities are ready while the rebuild branch still runs); 2: the rebuilt rollouts of the
// work list (grid.y-stride over it), after the rebuild branch joined.
// TF slots per CTA (see k_density); 40 registers at 48 resident warps per SM for every TF.
// The slot window (own_lo, own_n) of a domain-decomposition launch is a runtime tile offset;
// the same offset in every launch measures 3.9 % faster on C3 than a specialised offset-free
// instantiation (A/B on one box; its list loop is 8 SASS shorter, but the kernel is slower).
template <int TF, bool PP>
__global__ void __launch_bounds__(TF, SPH_FORCE_MINB * TILE / TF) k_force(DevParams P, DevPtrs D,
                                                                          float damping, int mode) {
    pdl_wait();
    pdl_trigger();
    const int tile = P.own_lo / TF + (int)blockIdx.x;
    if (mode == 2) {
        const int count = *D.rcount;
        for (int w = blockIdx.y; w < count; w += gridDim.y)
            force_tile<TF, true, PP>(P, D, damping, D.rlist[w], tile);
        return;
    }
    // snake order: k_density walks the rollouts first to last, k_force last to first, so the
    // first force CTAs find the rollouts k_density touched last still in L2
    const int b = P.snake ? (int)gridDim.y - 1 - (int)blockIdx.y : (int)blockIdx.y;
    if (mode == 1 && D.rs[b].need_rebin) return;   // CTA-uniform
    force_tile<TF, true, PP>(P, D, damping, b, tile);
    prefetch_ahead<true>(P, D, TF, P.pf_f, P.snake != 0);
}

// ---------------------------------------------------------------------------------------
// Ghost kinematics, Eq. kinematicghost, in fp64 from the fp64 body state.
// ---------------------------------------------------------------------------------------
// body[6], body[7] = cos(theta), sin(theta) (computed once per rollout)
// The body-frame loads of GU ghosts per thread are issued together before any store (restrict
// pointers, body state in registers): the loop is one L2 round trip per GU ghosts instead of one
// per ghost (k_body is a latency chain; same arithmetic, same bits).
constexpr int GU = 4;
__device__ __forceinline__ void ghost_update(const DevParams& P, const DevPtrs& D, int b,
                                             const double* body, int tid, int nthr) {
    const double c = body[6], s = body[7];
    const double r0 = body[0], r1 = body[1], v0 = body[3], v1 = body[4], w = body[5];
    const double2* __restrict__ gb = D.ghost_b;
    float4* __restrict__ gst = D.gst + (size_t)b * P.G;
    float2* __restrict__ glo = D.glo + (size_t)b * P.G;
    float2* __restrict__ garm = D.garm + (size_t)b * P.G;
    for (int g0 = tid; g0 < P.G; g0 += GU * nthr) {
        double2 q[GU];
#pragma unroll
        for (int k = 0; k < GU; ++k) {
            const int g = g0 + k * nthr;
            if (g < P.G) q[k] = __ldg(gb + g);
        }
#pragma unroll
        for (int k = 0; k < GU; ++k) {
            const int g = g0 + k * nthr;
            if (g >= P.G) break;
            const double ax = c * q[k].x - s * q[k].y, ay = s * q[k].x + c * q[k].y;
            const double wx = ax + r0, wy = ay + r1;
            const double vx = v0 - w * (wy - r1);
            const double vy = v1 + w * (wx - r0);
            const float hx = (float)wx, hy = (float)wy;
            gst[g] = make_float4(hx, hy, (float)vx, (float)vy);
            glo[g] = make_float2((float)(wx - (double)hx), (float)(wy - (double)hy));
            garm[g] = make_float2((float)(wx - r0), (float)(wy - r1));
        }
    }
}

// First stage of the body reduction of large tanks: CTA (s, b) sums the fixed chunk s of rollout
// b's per-warp partials (thread-strided, then a fixed-order tree) into part2[b][s].
constexpr int BRED_T = 256;
__global__ void __launch_bounds__(BRED_T) k_body_reduce(DevParams P, DevPtrs D) {
    __shared__ double4 red[BRED_T];
    const int b = blockIdx.y, sidx = blockIdx.x;
    if (D.rs[b].frozen) return;   // CTA-uniform
    const int chunk = (P.npart + P.bsplit - 1) / P.bsplit;
    const int t0 = sidx * chunk, t1 = min(t0 + chunk, P.npart);
    double4 s = make_double4(0, 0, 0, 0);
    for (int t = t0 + threadIdx.x; t < t1; t += BRED_T) {
        const double4 q = D.part[(size_t)b * P.npart + t];
        s.x += q.x;
        s.y += q.y;
        s.z += q.z;
        s.w = fmax(s.w, q.w);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = BRED_T / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double4 a = red[threadIdx.x], c = red[threadIdx.x + w];
            red[threadIdx.x] = make_double4(a.x + c.x, a.y + c.y, a.z + c.z, fmax(a.w, c.w));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) D.part2[(size_t)b * P.bsplit + sidx] = red[0];
}

// ---------------------------------------------------------------------------------------
// Body: fixed-order fp64 reduction of the CTA partials, Eq. tankdynamics
//   m rddot = -sum G + (u_x, u_y),  J thddot = sum (r_g - r) x (-G) + tau,
// symplectic Euler, status, rebuild policy, then ghosts for the next substep.
// ---------------------------------------------------------------------------------------
// blockDim.x = a power of two <= 1024, chosen from N only (so the reduction order, and hence
// the bits, never depend on the batch size).
// Body step of rollout b by the CTA: fixed-order fp64 reduction of the per-warp partials over
// the first nt threads (nt = k_body's block size, chosen from N only, so the bits never depend on
// the launch shape), Newton-Euler kick-then-drift, status, parity flips, rebuild decision, then
// the ghosts of the next substep by every thread.  red: shared memory [>= nt].  CTA-uniform.
// ghosts_here = 0 (large tanks, ghost_split): the ghost update of the next substep is left to
// k_ghosts, spread over many CTAs (cos / sin of theta handed over in D.body_cs)
__device__ __forceinline__ void body_step(const DevParams& P, const DevPtrs& D, int b, int pin,
                                          float ghost_angle0, double4* red, int nt, int ghosts_here = 1) {
    RolloutState* rs = D.rs + b;
    __shared__ double sbody[8];
    // thread 0's state loads, all issued before the reduction (independent; they complete while
    // the partials are summed) -- the serial part below then touches only registers
    double bd[6];
    float uu[3];
    int r_sp = 0, r_ip = 0, r_nr = 0, r_reb = 0, r_status = 0;
    if (threadIdx.x == 0) {
        const double* body = D.body + (size_t)b * 6;
        const float* u = D.u_cur + (size_t)b * 3;
#pragma unroll
        for (int c = 0; c < 6; ++c) bd[c] = body[c];
#pragma unroll
        for (int c = 0; c < 3; ++c) uu[c] = u[c];
        r_sp = rs->sp;
        r_ip = rs->ip;
        r_nr = rs->need_rebin;
        r_reb = rs->rebuilds;
        r_status = rs->status;
    }
    double4 s = make_double4(0, 0, 0, 0);
    const int np = P.bsplit > 1 ? P.bsplit : P.npart;
    const double4* part = P.bsplit > 1 ? D.part2 + (size_t)b * P.bsplit : D.part + (size_t)b * P.npart;
    if (threadIdx.x < nt)
        for (int t = threadIdx.x; t < np; t += nt) {
            const double4 q = part[t];
            s.x += q.x;
            s.y += q.y;
            s.z += q.z;
            s.w = fmax(s.w, q.w);
        }
    if (threadIdx.x < nt) red[threadIdx.x] = s;
    __syncthreads();
    // Tree over nt slots; slots >= np hold +0 (s starts at +0, so no slot is ever -0): the
    // levels whose upper halves are all such slots add exact zeros and are skipped (same bits).
    int w0 = nt / 2;
    while (w0 >= np && w0 > 1) w0 >>= 1;
    for (int w = w0; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            double4 a = red[threadIdx.x], c = red[threadIdx.x + w];
            red[threadIdx.x] = make_double4(a.x + c.x, a.y + c.y, a.z + c.z, fmax(a.w, c.w));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* body = D.body + (size_t)b * 6;
        const double4 f = red[0];
        double ax = 0.0, ay = 0.0;
        if (!pin) {
            ax = (f.x + (double)uu[0]) / P.m_body;
            ay = (f.y + (double)uu[1]) / P.m_body;
            const double ath = (f.z + (double)uu[2]) / P.J_body;
            bd[3] += P.dtd * ax;
            bd[4] += P.dtd * ay;
            bd[5] += P.dtd * ath;
            bd[0] += P.dtd * bd[3];
            bd[1] += P.dtd * bd[4];
            bd[2] += P.dtd * bd[5];
        }
        bool fin = true, big = false;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            body[c] = bd[c];
            sbody[c] = bd[c];
            fin = fin && isfinite(bd[c]);
            big = big || fabs(bd[c]) > 1e9;
        }
        if (!fin || big) {
            set_status(rs, fin ? 2 : 1, -1);   // (reads rs->step: this substep, before the increment)
            r_status = 1;
        }
        sincos(bd[2], &sbody[7], &sbody[6]);
        D.geom[b] = Geom{(float)bd[0], (float)bd[1], (float)(bd[2] + ghost_angle0),
                         (float)bd[3], (float)bd[4], {0.f, 0.f, 0.f}};
        const int nr = r_nr;
        rs->sp = r_sp ^ nr ^ 1;
        rs->ip = r_ip ^ nr;
        rs->rebuilds = r_reb + nr;
        // max over particles of |(x_i - x_i^build) - (r_n - r^build)| (from k_force) plus the
        // body's drift in this substep: a strict bound on every particle's displacement
        // relative to the body translation since the last rebuild (Verlet criterion)
        // uniform skin: d = that bound in metres.  Per-particle half-skins (B6): f.w is the
        // largest (|d_i| / hs_i)^2 and the body drift enters over the smallest half-skin, so
        // d >= rdisp = 0.98 whenever some |d_i| + drift may reach 0.98 hs_i
        const double drift = P.dtd * sqrt(bd[3] * bd[3] + bd[4] * bd[4]);
        const double d = sqrt(f.w) + (P.perpart ? drift / (double)P.hs_min : drift);
        const float disp = (float)d;
        rs->disp = disp;
        const int nrb = P.rebin_every ? 1 : (disp >= rs->rdisp ? 1 : 0);
        rs->need_rebin = nrb;
        if (nrb && !P.rebin_every) {   // the next substep rebuilds: adapt the skin (B5)
            const float sk = skin_adapt(P, rs->skin, rs->step + 1 - rs->last_reb);
            rs->skin = sk;
            skin_set(P, sk, &rs->rl2, &rs->rdisp);
            if (P.perpart) rs->rdisp = 0.98f;   // (B6: the bound is relative to hs_i)
            rs->last_reb = rs->step + 1;
        }
        rs->step += 1;
        if (r_status) rs->frozen = 1;
        D.body_cs[b] = make_double2(sbody[6], sbody[7]);
    }
    __syncthreads();
    if (ghosts_here) ghost_update(P, D, b, sbody, threadIdx.x, blockDim.x);
    __syncthreads();   // sbody / red reusable by the caller's next rollout
}

// blockDim.x = a power of two <= 1024, chosen from N only (so the reduction order, and hence
// the bits, never depend on the batch size).
__global__ void __launch_bounds__(1024) k_body(DevParams P, DevPtrs D, int pin,
                                               float ghost_angle0, int ghosts_here) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double4 red[];   // [blockDim.x]
    const int b = blockIdx.x;
    if (D.rs[b].frozen) return;        // CTA-uniform
    body_step(P, D, b, pin, ghost_angle0, red, blockDim.x, ghosts_here);
}

// Eq. kinematicghost for large tanks (G >= 4 x k_body's threads: C4 has 9,912 ghosts on one
// rollout, which one k_body CTA updated in ~10 us): grid (ceil(G / 256), B), the same
// ghost_update arithmetic from the body state and (cos, sin) k_body left -- identical bits.
constexpr int GH_T = 256;
__global__ void __launch_bounds__(GH_T) k_ghosts(DevParams P, DevPtrs D) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    double bd[8];
    const double* body = D.body + (size_t)b * 6;
#pragma unroll
    for (int c = 0; c < 6; ++c) bd[c] = body[c];
    const double2 cs = D.body_cs[b];
    bd[6] = cs.x;
    bd[7] = cs.y;
    ghost_update(P, D, b, bd, blockIdx.x * GH_T + threadIdx.x, gridDim.x * GH_T);
}

// ---------------------------------------------------------------------------------------
// Small batches (latency-bound: C1, P0, a single C2 tank): the whole substep loop of a slow
// tick in ONE cooperative launch.  Every phase of the multi-kernel path runs as a loop over
// virtual blocks of TILE threads separated by grid-wide barriers (cooperative groups), with
// the same per-particle, per-warp and per-rollout arithmetic -- so results are bitwise equal to
// the multi-kernel path (and independent of B).  No launch gaps, no per-kernel tails.
// ---------------------------------------------------------------------------------------
constexpr int COOP_T = TILE;
__global__ void __launch_bounds__(COOP_T, 2) k_coop(DevParams P, DevPtrs D, int n_sub,
                                                     float damping, int pin, float ghost_angle0,
                                                     int body_nt) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double4 red[COOP_T];
    const int G = gridDim.x;
    const int nt = P.ntile * P.B;                          // (tile, rollout) virtual blocks
    const int ncb = (P.ncell + TILE - 1) / TILE;
    for (int it = 0; it < n_sub; ++it) {
        int any = 0;
        for (int b = 0; b < P.B; ++b) any |= D.rs[b].need_rebin & (D.rs[b].frozen ^ 1);
        if (any) {   // grid-uniform: the counting sort of every rollout that needs it
            for (int v = blockIdx.x; v < nt; v += G) hash_blk(P, D, v % P.ntile, v / P.ntile);
            grid.sync();
            for (int v = blockIdx.x; v < P.nscan * P.B; v += G) scan_reduce_blk(P, D, v % P.nscan, v / P.nscan);
            grid.sync();
            for (int v = blockIdx.x; v < P.B; v += G) scan_tiles_blk(P, D, v, 0);
            grid.sync();
            for (int v = blockIdx.x; v < P.nscan * P.B; v += G) scan_down_blk(P, D, v % P.nscan, v / P.nscan);
            grid.sync();
            for (int v = blockIdx.x; v < nt; v += G) scatter_blk(P, D, v % P.ntile, v / P.ntile);
            grid.sync();
            for (int v = blockIdx.x; v < ncb * P.B; v += G) cellsort_blk(P, D, v % ncb, v / ncb);
            grid.sync();
            for (int v = blockIdx.x; v < nt; v += G) gather_blk(P, D, v % P.ntile, v / P.ntile);
            grid.sync();
        }
        // lists + densities of the rebuilt rollouts, densities of the others (disjoint rollouts)
        for (int v = blockIdx.x; v < nt; v += G) {
            const int b = v / P.ntile, i = (v % P.ntile) * TILE + threadIdx.x;
            const RolloutState* rs = D.rs + b;
            if (rs->frozen) continue;                      // CTA-uniform
            // coherent loads (NC = false): these rows were written earlier in this launch
            if (rs->need_rebin) {
                nlist_density_at<false>(P, D, b, i);
            } else if (i < P.N) {
                density_at<false>(P, D, b, i, D.pv[rs->sp] + (size_t)b * P.N);
            }
        }
        grid.sync();
        for (int v = blockIdx.x; v < nt; v += G) force_tile<TILE, false>(P, D, damping, v / P.ntile, v % P.ntile);
        grid.sync();
        for (int b = blockIdx.x; b < P.B; b += G)
            if (!D.rs[b].frozen) body_step(P, D, b, pin, ghost_angle0, red, body_nt);
        grid.sync();
    }
}

// ---------------------------------------------------------------------------------------
// Slow tick (multi-rate loop): sample y_k before u_k, set the ZOH
// input u_k from the table, tau from the PD law when pd != 0.
// ---------------------------------------------------------------------------------------
__global__ void k_tick(DevParams P, DevPtrs D, const float* __restrict__ u_seq,
                       const float* __restrict__ theta_ref, float* y, float* u_applied, int K,
                       int k, int pd, double Kp, double Kd) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= P.B) return;
    const double* body = D.body + (size_t)b * 6;
    const size_t bk = (size_t)b * K + k;
    for (int c = 0; c < 6; ++c) y[bk * 6 + c] = (float)body[c];
    float u0 = u_seq[bk * 3], u1 = u_seq[bk * 3 + 1], u2 = u_seq[bk * 3 + 2];
    if (pd) u2 = (float)(Kp * ((double)theta_ref[bk] - body[2]) - Kd * body[5]);
    D.u_cur[(size_t)b * 3] = u0;
    D.u_cur[(size_t)b * 3 + 1] = u1;
    D.u_cur[(size_t)b * 3 + 2] = u2;
    if (u_applied) {
        u_applied[bk * 3] = u0;
        u_applied[bk * 3 + 1] = u1;
        u_applied[bk * 3 + 2] = u2;
    }
}

// ---------------------------------------------------------------------------------------
// Host-boundary helpers: canonical-order import/export and ghost initialisation.
// ---------------------------------------------------------------------------------------
__global__ void k_import(DevParams P, DevPtrs D, int b0, const float4* __restrict__ in) {
    const int b = b0 + blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.N) return;
    const RolloutState* rs = D.rs + b;
    const size_t o = (size_t)b * P.N;
    D.pv[rs->sp][o + i] = in[i];
    D.id[rs->ip][o + i] = (uint32_t)i;
    D.skey[o + i] = 0u;   // canonical order = sorted by (cell 0, id): a valid start for k_resident
    D.aux[(size_t)b * P.NA + i] = make_float2(0.f, 0.f);
}

__global__ void k_export(DevParams P, DevPtrs D, int b, float4* out, float* rho) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.N) return;
    const RolloutState* rs = D.rs + b;
    const size_t o = (size_t)b * P.N;
    const uint32_t id = D.id[rs->ip][o + i];
    out[id] = D.pv[rs->sp][o + i];
    if (rho) rho[id] = D.aux[(size_t)b * P.NA + i].x;
}

// Domain decomposition (f2) exchange: the owned slots' new state (after k_force, before
// k_body) out to a caller buffer, and the gathered states of every slot back in (rollout 0).
__global__ void k_dd_export(DevParams P, DevPtrs D, float4* out) {
    const int i = P.own_lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.own_lo + P.own_n || i >= P.N) return;
    const RolloutState* rs = D.rs;
    out[i] = D.pv[rs->sp ^ rs->need_rebin ^ 1][i];
}

__global__ void k_dd_import(DevParams P, DevPtrs D, const float4* in) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.N) return;
    const RolloutState* rs = D.rs;
    D.pv[rs->sp ^ rs->need_rebin ^ 1][i] = in[i];
}

// Largest fluid speed of each rollout (sph_settle_until's convergence test).
__global__ void k_max_speed(DevParams P, DevPtrs D, float* out) {
    const int b = blockIdx.x;
    const RolloutState* rs = D.rs + b;
    const float4* pv = D.pv[rs->sp] + (size_t)b * P.N;
    float m = 0.0f;
    for (int i = threadIdx.x; i < P.N; i += blockDim.x) {
        const float4 v = pv[i];
        m = fmaxf(m, v.z * v.z + v.w * v.w);
    }
    m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));   // m >= 0
    __shared__ float sm[32];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float r = 0.0f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, sm[w]);
        out[b] = sqrtf(r);
    }
}

// clear_status = 0 (sph_set_body_state): only the pose-derived data (ghosts, float pose, rebuild
// flag) is refreshed; a failed rollout keeps its status, freeze and failure record.
__global__ void k_reset_rollout(DevParams P, DevPtrs D, int b0, float ghost_angle0, int clear_status) {
    const int b = b0 + blockIdx.x;
    RolloutState* rs = D.rs + b;
    __shared__ double sbody[8];
    if (threadIdx.x == 0) {
        rs->need_rebin = 1;
        if (clear_status) {
            rs->status = 0;
            rs->frozen = 0;
            rs->bad_step = -1;
            rs->bad_particle = -1;
        }
        rs->disp = 0.f;
        rs->skin = P.skin0;
        skin_set(P, P.skin0, &rs->rl2, &rs->rdisp);
        if (P.rebin_every) rs->rl2 = P.H2;
        if (P.perpart) rs->rdisp = 0.98f;
        rs->last_reb = rs->step;
        const double* body = D.body + (size_t)b * 6;
        for (int c = 0; c < 6; ++c) sbody[c] = body[c];
        sincos(body[2], &sbody[7], &sbody[6]);
        D.body_cs[b] = make_double2(sbody[6], sbody[7]);
        D.geom[b] = Geom{(float)body[0], (float)body[1], (float)(body[2] + ghost_angle0),
                         (float)body[3], (float)body[4], {0.f, 0.f, 0.f}};
    }
    __syncthreads();
    ghost_update(P, D, b, sbody, threadIdx.x, blockDim.x);
}

// Canonical cells of the current state (debug / parity, reading A19).
__global__ void k_debug_cells(DevParams P, DevPtrs D, int b, int* cells) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.N) return;
    const RolloutState* rs = D.rs + b;
    const size_t o = (size_t)b * P.N;
    const float4 x = D.pv[rs->sp][o + i];
    const Geom gm = D.geom[b];
    const float ox = __fsub_rn(gm.rx, P.half), oy = __fsub_rn(gm.ry, P.half);
    const uint32_t id = D.id[rs->ip][o + i];
    cells[2 * id] = cell_coord(x.x, ox, P.inv_C);
    cells[2 * id + 1] = cell_coord(x.y, oy, P.inv_C);
}

// Neighbour sets through the kernels' own enumeration (after a forced rebuild into the
// other buffer: reads pv[sp ^ 1], id[ip ^ 1]).
__global__ void k_debug_neighbours(DevParams P, DevPtrs D, int b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.N) return;
    const RolloutState* rs = D.rs + b;
    const size_t o = (size_t)b * P.N;
    const int cur = rs->sp ^ 1, ic = rs->ip ^ 1;
    const float4* pv = D.pv[cur] + o;
    const uint32_t* id = D.id[ic] + o;
    const float4 xi = pv[i];
    const uint32_t me = id[i];
    int* cnt = D.dbg_cnt;
    int* idx = D.dbg_idx;
    int n0 = 0, n1 = 0, n2 = 0;
    for_fluid_candidates(P, D, b, i, [&](uint32_t j) {
        const float4 xj = pv[j];
        const float r2 = dist2(__fsub_rn(xi.x, xj.x), __fsub_rn(xi.y, xj.y));
        if (r2 < P.H2) {
            if (n0 < DBG_CAP) idx[(size_t)me * DBG_CAP + n0] = (int)id[j];
            ++n0;
        }
    });
    const Geom gm = D.geom[b];
    const float4* gst = D.gst + (size_t)b * P.G;
    for_ghost_candidates(P, gm, make_float2(xi.x, xi.y), P.ghost_K, P.wall_r2, [&](int g) {
        const float4 xg = gst[g];
        const float r2 = dist2(__fsub_rn(xi.x, xg.x), __fsub_rn(xi.y, xg.y));
        if (r2 < P.H2) {
            if (n1 < DBG_CAP) idx[((size_t)P.N + me) * DBG_CAP + n1] = g;
            ++n1;
        }
        if (r2 < P.h2) {
            if (n2 < DBG_CAP) idx[((size_t)2 * P.N + me) * DBG_CAP + n2] = g;
            ++n2;
        }
    });
    cnt[me] = n0;
    cnt[P.N + me] = n1;
    cnt[2 * P.N + me] = n2;
}

}  // namespace sph
