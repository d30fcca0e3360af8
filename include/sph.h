/* include/sph.h -- C ABI of the B200-native SPH fuel-sloshing hot path (libsphb200.so).
 *
 * The library advances the coupled spacecraft + fluid model of arXiv 2604.12505 (P:n = line n
 * of the paper text, PAPER.md):  Sigma: xdot = f(x,u), y = h(x,u)  (Eq. NLmodel),
 * f = Algorithm 1 integrated with first-order symplectic Euler, the
 * multi-rate sample / control loop of P:263 and P:325, for B independent rollouts at once
 * (batched ensemble) on one GPU.  Every step of the path runs in the library's sm_100a
 * kernels; the caller provides device memory (e.g. a torch tensor) and a CUDA stream.
 *
 * Conventions
 *  - SI units, 2-D: rho in kg/m^2, P in N/m.  Particle state is float32; body state is float64.
 *  - Particle data crosses the ABI in CANONICAL order (the order the caller supplied at init);
 *    internal sorting by cell is invisible.
 *  - Body state layout (6 doubles) = y = [r_x r_y theta rdot_x rdot_y thetadot].
 *  - Input u = [u_x u_y tau] in the world frame at the CoM.
 *  - Errors: every call returns sph_status; nothing throws or aborts across the ABI.
 *    Argument / configuration errors return SPH_EINVAL before any device work.
 *    Numerical failure is per rollout (status 1 non-finite, 2 |x| > 1e9, 3 particle left the
 *    grid = tunnelled, 4 resident path only: a CTA's halo outgrew its shared-memory window,
 *    i.e. more than ~8 particles per cell along a cell row -- a compression the weakly
 *    compressible fluid does not reach before blowing up): that rollout freezes, the others
 *    continue, calls return SPH_OK and sph_get_status reports it; SPH_EBLOWUP only if every
 *    rollout failed.
 *  - Ownership: the caller owns the device workspace and every host buffer; the library never
 *    frees them.  The context owns only CUDA handles (graphs, events) and small staging
 *    buffers for host-pointer calls.
 *  - Streams: all device work is enqueued on the context's stream; calls that return host data
 *    synchronise that stream.  One context per host thread; several contexts per process are
 *    allowed.
 *  - Determinism: identical inputs give bitwise identical outputs, independent of the number
 *    of rollouts in the batch and of a rollout's position in it.
 */
#ifndef SPH_H
#define SPH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPH_OK = 0,
    SPH_EINVAL = 1,   /* bad argument or configuration                      */
    SPH_ENOMEM = 2,   /* workspace too small / staging allocation failed     */
    SPH_ECUDA = 3,    /* CUDA runtime error (message in sph_last_error)      */
    SPH_EBLOWUP = 4,  /* every rollout has a non-zero numerical status       */
    SPH_ESTATE = 6    /* call not valid in the context's current state       */
} sph_status;

typedef struct sph_ctx sph_ctx;

/* Fluid parameters: Table 2 plus the readings of DESIGN.md. */
typedef struct {
    double rho0;        /* base density rho_0 (Eq. EOS)                        */
    double k;           /* stiffness k (Eq. EOS)                                           */
    double alpha;       /* artificial viscosity factor (Eq. viscous)           */
    double beta;        /* boundary viscosity factor (Eq. viscous_b2f)          */
    double gamma1;      /* ghost density correction (Eq. density_update), (0,1] */
    double eps;         /* epsilon of the viscous denominators, > 0                */
    double h;           /* smoothing length h > 0 (cubic support 2h, spiky support h)      */
    double mass;        /* fluid particle mass m > 0 (reading R1: rho0 s^2)                */
    double w_cb_const;  /* cubic-spline constant C in C/h^2 (reading A1: 5/(14 pi))        */
    double ghost_pressure_sign; /* -1 repulsive wall (reading A4), +1 literal Alg. 1       */
    double gravity[2];  /* external acceleration on the fluid, world frame (0 = zero-g)    */
    double clamp_negative_pressure; /* 0: Eq. EOS as printed (default); 1: P = max(k (rho -
                                       rho0), 0), the ablation of SURVEY 8(b) (E1)  */
} sph_fluid_params;

/* Rigid spacecraft: Table 1.  Tank = circle of radius tank_radius at the CoM. */
typedef struct {
    double m;            /* mass > 0                 */
    double J;            /* inertia > 0              */
    double tank_radius;  /* inner wall radius R > 0  */
} sph_body_params;

/* Time stepping.  rebin_every = 1 rebuilds the cell list and the neighbour lists every
 * substep; 0 rebuilds them only when a particle may have moved (relative to the body
 * translation) by 0.49 skin since the last rebuild.  Cells and lists are then 2h + skin wide
 * (Verlet skin).  The lists hold every particle within 2h + skin (float32 predicate, reading
 * A19) and the density / force sums are cut at 2h by the kernels' shape (W and grad W vanish
 * continuously there, B3), so both modes evaluate the same neighbour sums. */
typedef struct {
    double dt;                /* fast step > 0                                 */
    int substeps_per_sample;  /* n_sub = T_s / dt >= 1 (multi-rate)    */
    int rebin_every;          /* 1 = every substep, 0 = adaptive with skin     */
    double skin;              /* >= 0, only used when rebin_every == 0         */
    int rebuild_path;         /* 0 auto; 1 one CTA per rebuilding rollout in shared memory
                                 (needs (n_cells+1)*4 + 10*n_fluid bytes <= 200 KB, else
                                 SPH_EINVAL); 2 grid-wide multi-kernel counting sort        */
    int exec_path;            /* how a slow tick runs; every path computes
                                 the same substep (Algorithm 1):
                                 0 auto: 3 when B x 16 <= the SM count and the rollout fits
                                   (latency-bound single tanks), else 2 for B*N <= 65536,
                                   else 1;
                                 1 per-substep kernels, one CUDA graph per tick;
                                 2 one cooperative launch per tick (k_coop);
                                 3 rollout-resident clusters (1.5-1.9x the
                                   cooperative tick for single tanks, 0.45x path 1 on C3):
                                   one thread-block cluster per rollout
                                   keeps its particles in distributed shared memory for the
                                   whole tick (k_resident); SPH_EINVAL if it does not fit     */
    double skin_max;          /* 0: fixed skin.  > skin: adaptive skin per rollout (B5):
                                 at every rebuild the skin is scaled by sqrt(8 / I), I = substeps
                                 the previous lists lasted, within [skin, skin_max]; cells are
                                 2h + skin_max wide.  The lists hold every pair within the
                                 rollout's current 2h + skin, so the sums are unchanged.      */
    int skin_mode;            /* with skin_max > skin: 0 per-rollout adaptive skin (B5);
                                 1 per-particle half-skins (B6): at every rebuild
                                 particle i gets hs_i = clamp(20 dt |v_i - v_body|, skin / 2,
                                 skin_max / 2), pair (i, j) is listed within 2h + hs_i + hs_j,
                                 and the lists are rebuilt when some particle's displacement
                                 reaches 0.98 hs_i (exec_path 3: mode 0 only).                */
} sph_time_params;

/* PD attitude law tau_k = Kp (theta_ref_k - theta_k) - Kd thetadot_k, ZOH. */
typedef struct {
    double Kp, Kd;
    const float* theta_ref;   /* [B][K]; same memory space as the call's other pointers */
} sph_pd_attitude;

/* Bytes of device workspace needed for B rollouts of n_fluid + n_ghost particles. 0 on bad args. */
size_t sph_workspace_bytes(const sph_fluid_params* fp, const sph_body_params* bp,
                           const sph_time_params* tp, int n_fluid, int n_ghost, int n_rollouts);

/* Create a context for B = n_rollouts identical tanks (the benchmark scenario):
 * fluid_pv  host float[n_fluid][4] = (x, y, vx, vy) world frame, canonical order;
 * ghost_body_xy host double[n_ghost][2] = body-frame ghost positions (fixed),
 *           uniformly spaced on the wall circle in angular order;
 * body at rest at the origin, theta = 0.  cuda_stream = cudaStream_t (NULL = default).
 * d_workspace: device memory of at least sph_workspace_bytes(...) bytes, 256-B aligned. */
sph_status sph_init_tank(const sph_fluid_params* fp, const sph_body_params* bp,
                         const sph_time_params* tp, int n_fluid, const float* fluid_pv,
                         int n_ghost, const double* ghost_body_xy, int n_rollouts,
                         void* cuda_stream, void* d_workspace, size_t workspace_bytes,
                         sph_ctx** out);

/* Replace the particle state of one rollout (rollout = -1: all) from host float[n_fluid][4]
 * in canonical order; body (host double[6]) may be NULL to keep it.  Clears its status. */
sph_status sph_set_state(sph_ctx* ctx, int rollout, const float* fluid_pv, const double* body);

/* Set all body states from host double[B][6].  Ghosts and the cell grid follow the new pose; the
 * rollouts' numerical status (sph_get_status) is kept: a failed rollout stays frozen. */
sph_status sph_set_body_state(sph_ctx* ctx, const double* body);

/* Copy one rollout's particles to host float[n_fluid][4] (canonical order).  rho (nullable):
 * host float[n_fluid], the densities evaluated in the last substep. */
sph_status sph_get_particles(sph_ctx* ctx, int rollout, float* fluid_pv, float* rho);

/* Copy one rollout's ghost world state (Eq. kinematicghost at the current body state) to host
 * float[n_ghost][4] = (x, y, vx, vy). */
sph_status sph_get_ghosts(sph_ctx* ctx, int rollout, float* ghost_pv);

/* Apply n_substeps substeps of the symplectic-Euler map with u held (ZOH).  u: [B][3]
 * (device pointer if ptr_on_device, else host). */
sph_status sph_step(sph_ctx* ctx, const float* u, int n_substeps, int ptr_on_device);

/* Multi-rate rollout (dataset D_N of Eq. dataset): for k < K sample
 * y_k = y(k T_s) BEFORE applying u_k, set u_k = u_seq[b][k] (tau overridden by the PD law when
 * pd != NULL), then run n_sub substeps.  u_seq [B][K][3], y_out [B][K][6], u_applied [B][K][3]
 * (nullable), all float32, device pointers if ptr_on_device else host. */
sph_status sph_rollout_batch(sph_ctx* ctx, const float* u_seq, int K, const sph_pd_attitude* pd,
                             float* y_out, float* u_applied, int ptr_on_device);

/* Current body states, host double[B][6] (P:70 output y). */
sph_status sph_get_body_state(sph_ctx* ctx, double* out);

/* Damped settling (reading A17): n_steps substeps with the body pinned at rest and the
 * fluid velocities multiplied by `damping` after each substep. */
sph_status sph_settle(sph_ctx* ctx, double damping, int n_steps);

/* P:323-324, "allowed to evolve without external actuation until their velocities converge to
 * zero": sph_settle in chunks of check_every substeps, each followed by the test, until every
 * rollout's largest fluid speed is below v_tol (m/s) or max_steps substeps were taken (at least
 * one chunk runs: a spawn starts at rest).  steps_done (nullable): substeps taken;
 * max_speed (nullable, host float[B]): the final largest speed per rollout.  Synchronises.
 * Errors: SPH_EINVAL bad arguments; SPH_ECUDA launch failure. */
sph_status sph_settle_until(sph_ctx* ctx, double damping, double v_tol, int max_steps,
                            int check_every, int* steps_done, float* max_speed);

/* Per-rollout numerical status (host int32[B]); bad_step (host int64[B], nullable) = substep
 * index of the failure; bad_particle (host int32[B], nullable) = canonical particle id. */
sph_status sph_get_status(sph_ctx* ctx, int32_t* rollout_status, int64_t* bad_step,
                          int32_t* bad_particle);

/* Parity / debug (reading A19).  Canonical float32 cell (c_x, c_y) of every particle of one
 * rollout at the current state: o = float(r_body) - half, c = floor((x - o) * inv), no FMA.
 * cells host int32[n_fluid][2]; grid host float[4] = (o_x, o_y, inv, cell side). */
sph_status sph_debug_cells(sph_ctx* ctx, int rollout, int32_t* cells, float* grid);

/* Neighbour sets of one rollout at the current state, from the cell-list enumeration the
 * kernels use: NF(i) (fluid, |r|^2 < (2h)^2, j != i), NG2(i) (ghosts within 2h), NG1(i)
 * (ghosts within h); float32 predicates, no FMA.  CSR in canonical order with ascending ids:
 * *_off host int64[n_fluid+1], *_idx host int32[cap].  Returns SPH_ENOMEM if cap too small. */
sph_status sph_debug_neighbours(sph_ctx* ctx, int rollout, int64_t* nf_off, int32_t* nf_idx,
                                int64_t nf_cap, int64_t* g2_off, int32_t* g2_idx,
                                int64_t g2_cap, int64_t* g1_off, int32_t* g1_idx,
                                int64_t g1_cap);

/* Kernel timing (CUDA events on the context stream, no graph): runs n_substeps substeps with
 * u held and writes the average device time per launch in ms of each kernel into
 * ms[SPH_NUM_TIMERS] (order: see SPH_TIMER_* below). */
enum {
    SPH_TIMER_REBUILD = 0,  /* cell sort + neighbour lists of the rollouts that need it (small
                               path: also their densities)                                 */
    SPH_TIMER_DENSITY = 1, SPH_TIMER_FORCE = 2, SPH_TIMER_BODY = 3, SPH_TIMER_SUBSTEP = 4,
    SPH_TIMER_SORT = 5,     /* the cell-sort part of SPH_TIMER_REBUILD (plan + sort kernels)     */
    SPH_NUM_TIMERS = 6
};
sph_status sph_profile_substeps(sph_ctx* ctx, int n_substeps, float* ms);

/* Live kernel timing inside sph_rollout_batch (the production path, CUDA graph included).
 * every > 0: the tick graph is re-captured with event-record nodes around the density launch,
 * the force launch(es) and the whole substep of every `every`-th substep; after each tick the
 * host synchronises the context stream (one host round trip per tick) and adds the elapsed
 * times to accumulators.  every = 0 disables it (graph re-captured without the nodes).
 * sph_get_live_timing writes the sums in ms over the sampled substeps into
 * ms_sum[SPH_NUM_LIVE] (order SPH_LIVE_*) and their count into *n_samples (nullable);
 * reset != 0 zeroes the accumulators afterwards.  In the small-rollout path the density and
 * the force launches overlap the rebuild branch, so these are in-situ durations; the forces of
 * the rebuilt rollouts run on that branch concurrently with the others', and the force time is
 * the union of the two launches' active intervals. */
/* Resident path (exec_path 3): each tick is ONE kernel launch (k_resident: every substep of the
 * tick for every rollout); every > 0 records CUDA events around every such launch, and
 * ms_sum[SPH_LIVE_TICK] sums their durations (n_samples counts ticks; the other slots stay 0). */
enum { SPH_LIVE_DENSITY = 0, SPH_LIVE_FORCE = 1, SPH_LIVE_SUBSTEP = 2, SPH_LIVE_TICK = 3, SPH_NUM_LIVE = 4 };
sph_status sph_set_live_timing(sph_ctx* ctx, int every);
sph_status sph_get_live_timing(sph_ctx* ctx, double* ms_sum, int64_t* n_samples, int reset);

/* Linearization (P:259 item 2 "exact and efficient computation of the Jacobian
 * of the state transition function", P:408-413 eigenvalues of the linearized open-loop system).
 * Jacobians of the continuous-time model f(x, u) (Eq. NLmodel; Algorithm 1 l.1-8,
 * Eq. tankdynamics) at rollout `rollout`'s current state:
 *   x = [pos (n_fluid x 2, canonical id order), vel (n_fluid x 2), r_x, r_y, theta, rd_x, rd_y,
 *        thd], n_x = 4 n_fluid + 6;  u = (u_x, u_y, tau);
 *   f = [vel, a, rd, thd, (F_b + u_xy) / m_B, (T_b + tau) / J].
 * f is affine in u, so A and B do not depend on the input.  Forward-mode (tangent-linear)
 * differentiation in float64 on the GPU, one unit seed per column; the operating point is the
 * float32 state converted exactly to float64; neighbour sets are the float64 predicates
 * |x_i - x_j|^2 < (2h)^2, |x_i - x_g|^2 < (2h)^2 / h^2 at that point (held fixed: kernel values
 * and gradients vanish at the support).
 * A: n_x x n_x, B: n_x x 3, row-major float64, caller-owned; device pointers (ctx stream) if
 * ptr_on_device, else host (the call synchronises).  Device scratch of O(n_fluid) (+ 8 n_x^2
 * bytes for host pointers) is kept by the context for later calls (freed by sph_destroy).
 * Errors: SPH_EINVAL bad arguments; SPH_ENOMEM more than 48 fluid neighbours or ghosts around
 * one particle; SPH_ECUDA allocation / launch failure. */
sph_status sph_jacobian(sph_ctx* ctx, int rollout, double* A, double* B, int ptr_on_device);

/* Eigenvalues of a dense real n x n float64 matrix (Figs. 5-6: spectra of the
 * linearized systems), by the GPU library eigensolver (cuSOLVER Xgeev, no eigenvectors) on the
 * context stream.  A: column- or row-major does not matter for eigenvalues (A and A^T share
 * them); it is overwritten.  w: n complex values as (re, im) double pairs.  A and w are device
 * pointers if ptr_on_device, else host (copied in / out; the call synchronises).
 * Errors: SPH_EINVAL bad arguments; SPH_ECUDA solver failure (message in sph_last_error). */
sph_status sph_eigenvalues(sph_ctx* ctx, int n, double* A, double* w, int ptr_on_device);

/* Analytic estimate of the wall correcting factor gamma1 (Eq. gamma1; SURVEY 8(f)
 * f4) on rollout `rollout`'s current state:
 *   gamma1_i = (rho_target / m - sum_f W_cb(r_if)) / sum_g W_cb(r_ig)
 * (printed denominator subscript i_b read as the ghost sum, reading G1).  Sums as in Eq.
 * density_update, self term included in the fluid sum, float32 support predicate
 * (reading A19) over every fluid particle and ghost (O(n_fluid^2) brute force: a calibration
 * utility, not a per-step call).  Outputs (host pointers, each may be NULL; the call
 * synchronises): gamma1_i [n_fluid] float32 in canonical id order (NaN where no ghost lies within
 * 2h); sums [n_fluid][2] float32 = (sum_f W, sum_g W) / (C/h^2); gamma1_wall = the estimate of
 * the whole wall layer, sum of the numerators over sum of the denominators of the particles with
 * a ghost within 2h (float64; NaN if there is none).
 * Errors: SPH_EINVAL bad arguments (rho_target <= 0); SPH_ECUDA launch / allocation failure. */
sph_status sph_gamma1_estimate(sph_ctx* ctx, int rollout, double rho_target, float* gamma1_i,
                               float* sums, double* gamma1_wall);

/* ---- Spatial domain decomposition of one tank ----------------------------
 * Replicated-data decomposition over W processes (one GPU each): every process holds the whole
 * tank, sorts it by cell (identically: the rebuild is deterministic) and computes density,
 * forces and integration only for its slab of the cell-sorted slots, [slot_lo, slot_hi) -- a
 * band of cell rows.  Per substep three phases, with the caller all-gathering three
 * caller-owned device buffers between them (NCCL all-gather over NVLink in
 * paper_2604_12505_b200/parallel.py):
 *   phase 0: input u (host float[3], NULL: keep), rebuild if due, densities of the owned slots
 *            -> aux_io[slot] = (rho, P/rho^2)                          (float2 [n_fluid])
 *   (all-gather aux_io)
 *   phase 1: forces + symplectic Euler of the owned slots -> state_io[slot] = new (x, y, vx, vy)
 *            (float4 [n_fluid]) and part_io[warp] = body partials of the owned warps
 *            (double4 [8 ceil(n_fluid / 256)]: F_x, F_y, T, max displacement^2)
 *   (all-gather state_io and part_io)
 *   phase 2: import the gathered state, body reduction (fixed order over every warp) and body
 *            step, identical on every process.
 * Every slot's arithmetic is the single-GPU path's, and the body sum runs in the same order, so
 * the decomposed trajectory is bitwise identical to the undecomposed one.  Requirements: one
 * rollout; slot_lo and slot_hi multiples of SPH_DD_ALIGN (slot_hi may be n_fluid).  Setting a
 * domain switches the context to the per-substep kernel path (no cooperative tick) for good.
 * Slot order: the cell-sorted order of the last rebuild (sph_get_particles returns canonical
 * order).  Numerical-failure status stays local to the process whose slot failed.
 * Errors: SPH_EINVAL bad arguments / range; SPH_ECUDA launch failure. */
#define SPH_DD_ALIGN 1024
sph_status sph_set_domain(sph_ctx* ctx, int slot_lo, int slot_hi);
sph_status sph_dd_phase(sph_ctx* ctx, int phase, const float* u, void* aux_io, void* state_io,
                        void* part_io);

/* ---- LPV surrogate identification (paper Sec. 4, Sec. 5.3
 * P:423-446).  Context-free calls on DEVICE pointers, enqueued on `stream` (a cudaStream_t, NULL =
 * the legacy default stream); they do not synchronise.
 * Model: self-scheduled LPV-SS with affine scheduling (Eqs. surrogate_form, LPVparametrization),
 * n_x = 4, n_u = 3, n_y = 3, n_p = 1, D = 0, scheduling map [x; u] -> 4 tanh -> 4 tanh -> 1
 * (P:438-440).  Parameters of restart r: params[r] = [theta (SPH_LPV_NTHETA), x0 (S x 4)], float64,
 * theta = A0 (4x4) B0 (4x3) C0 (3x4) A1 (4x4) B1 (4x3) C1 (3x4) W1 (4x7) b1 (4) W2 (4x4) b2 (4)
 * W3 (1x4) b3 (1), row-major (137 values: SPEC's count; the paper prints 130, reading LPV1). */
#define SPH_LPV_NTHETA 137

/* Device scratch bytes of sph_lpv_eval for R restarts, S sequences of K samples (0 on bad sizes). */
size_t sph_lpv_scratch_bytes(int R, int S, int K);

/* Objective and gradient of Eq. surrogate_optimization for R parameter sets at once:
 *   F_r = 1/S sum_s 1/K sum_k ||y_sk - y^_sk||^2 + sigma2/2 ||theta_r||^2
 *         + sigmax/2 sum_s ||x0_rs||^2                  (Eqs. pem, regularization; reading LPV3)
 * u: [S][K][3], y: [S][K][3] float32 (the scaled, normalised dataset); obj [R], grad [R][137 + 4S]
 * (same layout as params; reverse-mode gradient), yhat [R][S][K][3] float32: each may be NULL
 * (y may be NULL when obj and grad are).  scratch: >= sph_lpv_scratch_bytes(R, S, K) device bytes.
 * Errors: SPH_EINVAL bad sizes / pointers / weights; SPH_ECUDA launch failure. */
sph_status sph_lpv_eval(int R, int S, int K, const double* params, const float* u, const float* y,
                        double sigma2, double sigmax, double* obj, double* grad, float* yhat,
                        void* scratch, size_t scratch_bytes, void* stream);

/* One Adam step on R x n float64 parameters in place: m, v moment buffers (zero at t = 1),
 * t >= 1 the step number (bias correction), mask [n] uint8 or NULL: 0 freezes that parameter of
 * every restart.  Errors: SPH_EINVAL bad arguments; SPH_ECUDA launch failure. */
sph_status sph_lpv_adam(int R, int n, double* w, const double* g, double* m, double* v, double lr,
                        double beta1, double beta2, double eps, int t, const uint8_t* mask,
                        void* stream);

/* Per-rollout counters (host arrays of B, nullable): substeps taken and cell-list / neighbour-
 * list rebuilds performed (with rebin_every = 0 rebuilds happen only when the displacement
 * bound requires them). */
sph_status sph_get_counters(sph_ctx* ctx, int64_t* steps, int32_t* rebuilds);

/* Number of our kernel launches one substep issues (for the bench's gpu_launches count);
 * 0 when the context runs small batches as one cooperative launch per tick (or per sph_step /
 * sph_settle call) instead of per-substep kernels. */
int sph_launches_per_substep(const sph_ctx* ctx);

/* Exact number of our kernel launches one slow tick of sph_rollout_batch issues: 1 + n_sub x
 * (launches per substep) on the per-substep path (sampling kernel + graph), 2 for the
 * cooperative tick, 1 for the resident path (sampling fused into k_resident); 0 on a NULL ctx. */
int sph_launches_per_tick(const sph_ctx* ctx);

/* Execution path the context runs (1, 2 or 3, see sph_time_params.exec_path; 0 on NULL) and, for
 * the resident path, its shape: CTAs per rollout (cluster size), threads per CTA, slots per CTA
 * and dynamic shared memory per CTA in bytes (any pointer may be NULL). */
int sph_exec_path(const sph_ctx* ctx, int* cluster_ctas, int* threads, int* slots_per_cta,
                  int* smem_bytes);

/* Sizes of the context (any pointer may be NULL). */
void sph_get_sizes(const sph_ctx* ctx, int* n_fluid, int* n_ghost, int* n_rollouts,
                   int* n_cells);

/* Last error message of this context (or of the last failed sph_init_tank when ctx == NULL). */
const char* sph_last_error(const sph_ctx* ctx);

/* Destroy the context (CUDA handles only; the workspace stays the caller's). */
void sph_destroy(sph_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SPH_H */
