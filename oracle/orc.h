/* oracle/orc.h -- plain, slow, float64 CPU oracle of the SPH fuel-sloshing substep.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header or constant with the CUDA path (paper_2604_12505_b200/csrc, include/sph.h).
 *
 * Every function follows the paper text step by step (P:n = PAPER.md line n) in the order
 * of Algorithm 1 and the readings listed in DESIGN.md ("Readings").
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double rho0, k, alpha, beta, gamma1, eps, h, mass;
    double w_cb_const;            /* 5/(14 pi) normalised (reading A1) */
    double ghost_pressure_sign;   /* -1: repulsive wall (reading A4)    */
    double gx, gy;                /* external acceleration on the fluid */
    double m_body, J_body, R;     /* Table 1 */
    double dt;                    /* fast step */
    double clamp_negative_pressure; /* 1: P = max(k (rho - rho0), 0) (ablation); 0: Eq. EOS */
} orc_params;

/* Kernels. r = |x|. dW = dW/dr. */
double orc_W_cb(const orc_params* p, double r);
double orc_dW_cb(const orc_params* p, double r);
double orc_W_s3(const orc_params* p, double r);
double orc_dW_s3(const orc_params* p, double r);

/* Neighbour sets NF(i) = {j != i : |r_ij|^2 < (2h)^2} as CSR with ascending ids.
 * use_cells = 0: O(N^2) brute force; 1: cell list.  Returns number of pairs, or -1 if
 * cap too small.  off[n+1]. */
int64_t orc_neighbours(const orc_params* p, int n, const double* pos, int use_cells,
                       int64_t* off, int32_t* idx, int64_t cap);

/* Eq. kinematicghost: world positions / velocities of the ghosts. */
void orc_ghosts(int ng, const double* gB, const double* body, double* gpos, double* gvel);

/* Eqs. density_update + EOS.  rho[n], P[n]. */
/* The two kernel sums of Eq. density_update, in units of W_cb (m = 1, gamma1 = 1
 * kept apart): sf[i] = sum over fluid j (self included) W_cb(r_ij), sg[i] = sum over ghosts
 * W_cb(r_ig).  Ingredients of the gamma1 estimate, Eq. gamma1. */
void orc_density_parts(const orc_params* p, int n, const double* pos, int ng, const double* gpos,
                       double* sf, double* sg);
void orc_density(const orc_params* p, int n, const double* pos, int ng, const double* gpos,
                 double* rho, double* P);

/* Eqs. momentum, viscous, pressure_b2f, viscous_b2f, tankdynamics and
 * Algorithm 1 l.8.  acc[n][2] fluid accelerations; Fb[2], Tb: fluid->body
 * force and torque (WITHOUT the external input u). */
void orc_forces(const orc_params* p, int n, const double* pos, const double* vel,
                const double* rho, const double* P, int ng, const double* gpos,
                const double* gvel, const double* body, double* acc, double* Fb, double* Tb);

/* One fast substep (Algorithm 1 + symplectic Euler kick-then-drift).
 * body[6] = r_x r_y theta rd_x rd_y thd.  u[3] = u_x u_y tau.
 * damping: fluid velocities multiplied by it after the step (settling, reading A17; 1 = off).
 * pin_body: 1 keeps the body at rest (settling).  rho_out nullable.
 * Returns 0 ok, 1 non-finite, 2 |x| > 1e9 (S:267 reading). */
int orc_step(const orc_params* p, int n, double* pos, double* vel, int ng, const double* gB,
             double* body, const double* u, double damping, int pin_body, double* rho_out);

/* Multi-rate rollout (Eq. dataset): for k < K: y_k = body (sampled
 * before u_k is applied), u_k from u_seq (ZOH); if theta_ref != NULL the torque is the PD law
 * tau_k = Kp (theta_ref_k - theta_k) - Kd thd_k. Then n_sub substeps.
 * Returns 0 or the first failing status; *bad_step = global substep index of failure. */
int orc_rollout(const orc_params* p, int n, double* pos, double* vel, int ng, const double* gB,
                double* body, int K, int n_sub, const double* u_seq, const double* theta_ref,
                double Kp, double Kd, double* y_out, double* u_applied, int64_t* bad_step);

/* ---- linearization -------------------------------- */
/* Continuous-time f(x, u) of Sigma: x = [pos (n x 2), vel (n x 2), r_x, r_y, theta,
 * rd_x, rd_y, thd] (n_x = 4n + 6), u = (u_x, u_y, tau); xdot[n_x]. */
void orc_deriv(const orc_params* p, int n, const double* x, int ng, const double* gB,
               const double* u, double* xdot);
/* Central-difference Jacobian A = df/dx (n_x x n_x), B = df/du (n_x x 3), row-major, step
 * h_j = h_rel max(1, |x_j|) (SPEC linearization: h_rel = 1e-6). */
void orc_jacobian_fd(const orc_params* p, int n, const double* x, int ng, const double* gB,
                     const double* u, double h_rel, double* A, double* B);

/* ---- float32 parity predicates (reading A19), evaluated on given float32 values ----- */
/* Cell of each point: c_x = floor((x - o_x) * inv) with IEEE float32 ops, no contraction.
 * o = (float)body_r - half.  cells[n][2]. */
void orc_cells_f32(int n, const float* pos, float ox, float oy, float inv, int32_t* cells);
/* NF(i) with float32 predicate dx*dx + dy*dy < H2 (dx = xi - xj), ascending CSR. */
int64_t orc_neighbours_f32(int n, const float* pos, float H2, int64_t* off, int32_t* idx,
                           int64_t cap);
/* Ghost sets NG(i) = {g : |x_i - x_g|^2 < R2} float32 predicate, ascending CSR. */
int64_t orc_ghost_neighbours_f32(int n, const float* pos, int ng, const float* gpos, float R2,
                                 int64_t* off, int32_t* idx, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
