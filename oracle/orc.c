/* oracle/orc.c -- plain, slow, float64 CPU oracle of the SPH fuel-sloshing substep.
 *
 * TEST INFRASTRUCTURE ONLY (see orc.h).  Compiled with -O2 -ffp-contract=off, no intrinsics,
 * no SIMD, single-threaded.  Written from the paper (P:n = PAPER.md line n):
 *   kernels            Eq. cubicspline P:268-270 (constant: reading A1), Eq. spiky3
 *   neighbour sets     footnote P:135 (only particles inside the support contribute)
 *   ghosts             Eq. kinematicghost
 *   density            Eq. density_update P:180-182 (self term included, "all particles")
 *   pressure           Eq. EOS P:149-151 (no clamp, reading A10)
 *   fluid forces       Eq. momentum, Eq. viscous, gradient P:153-155
 *   wall forces        Eqs. pressure_b2f/f2b P:188-194 (sign: reading A4),
 *                      viscous_b2f/f2b P:197-203 (rho_g := rho_f, m_g := m_f)
 *   body               Eq. tankdynamics
 *   acceleration       Algorithm 1 l.8 P:248
 *   integrator         symplectic Euler, kick then drift (reading A11)
 *   multi-rate loop    P:263; PD law P:366-374; dataset Eq. P:97-100
 * Sums run over neighbours in ascending particle id (self term first).
 */
#include "orc.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------------------ */
/* Kernels                                                                    */
/* ------------------------------------------------------------------------------------ */
double orc_W_cb(const orc_params* p, double r) {
    double h = p->h, q = r / h, c = p->w_cb_const / (h * h);
    if (q <= 1.0) return c * ((2.0 - q) * (2.0 - q) * (2.0 - q) - 4.0 * (1.0 - q) * (1.0 - q) * (1.0 - q));
    if (q < 2.0) return c * (2.0 - q) * (2.0 - q) * (2.0 - q);
    return 0.0;
}

/* d W_cb / d r = (C / h^3) d f / d q */
double orc_dW_cb(const orc_params* p, double r) {
    double h = p->h, q = r / h, c = p->w_cb_const / (h * h * h);
    if (q <= 1.0) return c * (-3.0 * (2.0 - q) * (2.0 - q) + 12.0 * (1.0 - q) * (1.0 - q));
    if (q < 2.0) return c * (-3.0 * (2.0 - q) * (2.0 - q));
    return 0.0;
}

double orc_W_s3(const orc_params* p, double r) {
    double h = p->h;
    if (r <= h) return 10.0 / (M_PI * pow(h, 5)) * (h - r) * (h - r) * (h - r);
    return 0.0;
}

double orc_dW_s3(const orc_params* p, double r) {
    double h = p->h;
    if (r < h) return -30.0 / (M_PI * pow(h, 5)) * (h - r) * (h - r);
    return 0.0;
}

/* nabla_i W_ij = W'(|r_ij|) r_ij / |r_ij|; zero vector at r = 0 (reading A8) */
static void grad(double dW, double rx, double ry, double r, double* gx, double* gy) {
    if (r > 0.0) {
        *gx = dW * rx / r;
        *gy = dW * ry / r;
    } else {
        *gx = 0.0;
        *gy = 0.0;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Neighbour search: a plain uniform grid (cell side = query radius) or brute force.        */
/* Results are sorted ascending so every sum runs in ascending id.                          */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    double x0, y0, cs;
    int nx, ny, n;
    int* start; /* nx*ny+1 */
    int* items; /* n */
} grid_t;

static void grid_build(grid_t* g, int n, const double* pts, double cs) {
    double xmin = 0, xmax = 0, ymin = 0, ymax = 0;
    int i;
    for (i = 0; i < n; i++) {
        double x = pts[2 * i], y = pts[2 * i + 1];
        if (i == 0 || x < xmin) xmin = x;
        if (i == 0 || x > xmax) xmax = x;
        if (i == 0 || y < ymin) ymin = y;
        if (i == 0 || y > ymax) ymax = y;
    }
    g->n = n;
    g->cs = cs;
    g->x0 = xmin;
    g->y0 = ymin;
    double fx = (xmax - xmin) / cs + 1.0, fy = (ymax - ymin) / cs + 1.0;
    /* sparse point sets (e.g. a ghost ring): coarser cells are still correct for a query
       radius <= cell side (3 x 3 cells are scanned) */
    for (int k = 0; k < 40 && fx * fy > 4.0 * n + 4e6; k++) {
        g->cs *= 2.0;
        fx = (xmax - xmin) / g->cs + 1.0;
        fy = (ymax - ymin) / g->cs + 1.0;
    }
    if (n == 0 || !(fx * fy <= 4.0 * n + 4e6)) { /* degenerate / exploded: one cell */
        g->nx = 1;
        g->ny = 1;
        g->cs = INFINITY;
    } else {
        g->nx = (int)fx;
        g->ny = (int)fy;
    }
    int nc = g->nx * g->ny;
    g->start = (int*)calloc((size_t)nc + 1, sizeof(int));
    g->items = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int* cell = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (i = 0; i < n; i++) {
        int cx = 0, cy = 0;
        if (g->nx > 1 || g->ny > 1) {
            cx = (int)floor((pts[2 * i] - g->x0) / g->cs);
            cy = (int)floor((pts[2 * i + 1] - g->y0) / g->cs);
            if (cx < 0) cx = 0;
            if (cy < 0) cy = 0;
            if (cx >= g->nx) cx = g->nx - 1;
            if (cy >= g->ny) cy = g->ny - 1;
        }
        cell[i] = cy * g->nx + cx;
        g->start[cell[i] + 1]++;
    }
    for (i = 0; i < nc; i++) g->start[i + 1] += g->start[i];
    int* fill = (int*)malloc(sizeof(int) * (size_t)nc);
    memcpy(fill, g->start, sizeof(int) * (size_t)nc);
    for (i = 0; i < n; i++) g->items[fill[cell[i]]++] = i; /* ascending within a cell */
    free(fill);
    free(cell);
}

static void grid_free(grid_t* g) {
    free(g->start);
    free(g->items);
}

static void sort_ints(int* a, int m) { /* insertion sort: lists are short */
    for (int i = 1; i < m; i++) {
        int v = a[i], j = i - 1;
        while (j >= 0 && a[j] > v) {
            a[j + 1] = a[j];
            j--;
        }
        a[j + 1] = v;
    }
}

/* Indices k of pts with |q - pts_k|^2 < r2 (k != skip), ascending.  Returns count. */
static int grid_query(const grid_t* g, const double* pts, double qx, double qy, double r2,
                      int skip, int** buf, int* cap) {
    int m = 0;
    int cx0 = 0, cx1 = g->nx - 1, cy0 = 0, cy1 = g->ny - 1;
    if (isfinite(g->cs)) {
        cx0 = (int)floor((qx - g->x0) / g->cs) - 1;
        cx1 = cx0 + 2;
        cy0 = (int)floor((qy - g->y0) / g->cs) - 1;
        cy1 = cy0 + 2;
        if (cx0 < 0) cx0 = 0;
        if (cy0 < 0) cy0 = 0;
        if (cx1 > g->nx - 1) cx1 = g->nx - 1;
        if (cy1 > g->ny - 1) cy1 = g->ny - 1;
    }
    for (int cy = cy0; cy <= cy1; cy++)
        for (int cx = cx0; cx <= cx1; cx++) {
            int c = cy * g->nx + cx;
            for (int t = g->start[c]; t < g->start[c + 1]; t++) {
                int k = g->items[t];
                if (k == skip) continue;
                double dx = qx - pts[2 * k], dy = qy - pts[2 * k + 1];
                if (dx * dx + dy * dy < r2) {
                    if (m == *cap) {
                        *cap = *cap * 2 + 16;
                        *buf = (int*)realloc(*buf, sizeof(int) * (size_t)*cap);
                    }
                    (*buf)[m++] = k;
                }
            }
        }
    sort_ints(*buf, m);
    return m;
}

static int brute_query(int n, const double* pts, double qx, double qy, double r2, int skip,
                       int** buf, int* cap) {
    int m = 0;
    for (int k = 0; k < n; k++) {
        if (k == skip) continue;
        double dx = qx - pts[2 * k], dy = qy - pts[2 * k + 1];
        if (dx * dx + dy * dy < r2) {
            if (m == *cap) {
                *cap = *cap * 2 + 16;
                *buf = (int*)realloc(*buf, sizeof(int) * (size_t)*cap);
            }
            (*buf)[m++] = k;
        }
    }
    return m;
}

int64_t orc_neighbours(const orc_params* p, int n, const double* pos, int use_cells,
                       int64_t* off, int32_t* idx, int64_t cap) {
    double H = 2.0 * p->h;
    grid_t g;
    int bcap = 64;
    int* buf = (int*)malloc(sizeof(int) * (size_t)bcap);
    if (use_cells) grid_build(&g, n, pos, H);
    int64_t tot = 0;
    off[0] = 0;
    for (int i = 0; i < n; i++) {
        int m = use_cells ? grid_query(&g, pos, pos[2 * i], pos[2 * i + 1], H * H, i, &buf, &bcap)
                          : brute_query(n, pos, pos[2 * i], pos[2 * i + 1], H * H, i, &buf, &bcap);
        for (int t = 0; t < m; t++) {
            if (tot < cap) idx[tot] = buf[t];
            tot++;
        }
        off[i + 1] = tot;
    }
    if (use_cells) grid_free(&g);
    free(buf);
    return tot <= cap ? tot : -1;
}

/* ------------------------------------------------------------------------------------ */
/* Step 1: ghost kinematics, Eq. kinematicghost.                              */
/*   r_g = R(theta) r_g^B + r ;  rdot_g = rdot + thetadot x (r_g - r),                    */
/*   2-D cross  w x a = (-w a_y, w a_x).                                                  */
/* ------------------------------------------------------------------------------------ */
void orc_ghosts(int ng, const double* gB, const double* body, double* gpos, double* gvel) {
    double c = cos(body[2]), s = sin(body[2]);
    for (int g = 0; g < ng; g++) {
        double xb = gB[2 * g], yb = gB[2 * g + 1];
        gpos[2 * g] = c * xb - s * yb + body[0];
        gpos[2 * g + 1] = s * xb + c * yb + body[1];
        double ax = gpos[2 * g] - body[0], ay = gpos[2 * g + 1] - body[1];
        gvel[2 * g] = body[3] - body[5] * ay;
        gvel[2 * g + 1] = body[4] + body[5] * ax;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Steps 3-4: density (Eq. density_update) and pressure (Eq. EOS).   */
/*   rho_i = m_i ( sum_{i_f} W_cb(r_i,i_f) + gamma1 sum_{i_g} W_cb(r_i,i_g) ),            */
/*   the fluid sum includes i itself ("all particles"), cubic kernel.       */
/* ------------------------------------------------------------------------------------ */
void orc_density_parts(const orc_params* p, int n, const double* pos, int ng, const double* gpos,
                       double* sf, double* sg) {
    /* the two sums of Eq. density_update, formed as in orc_density below with the
     * mass and gamma1 factors left out */
    double H = 2.0 * p->h;
    grid_t gf, gg;
    grid_build(&gf, n, pos, H);
    grid_build(&gg, ng, gpos, H);
    int cap = 64;
    int* buf = (int*)malloc(sizeof(int) * (size_t)cap);
    for (int i = 0; i < n; i++) {
        double xi = pos[2 * i], yi = pos[2 * i + 1];
        double f = orc_W_cb(p, 0.0); /* self term */
        int m = grid_query(&gf, pos, xi, yi, H * H, i, &buf, &cap);
        for (int t = 0; t < m; t++) {
            int j = buf[t];
            double dx = xi - pos[2 * j], dy = yi - pos[2 * j + 1];
            f += orc_W_cb(p, sqrt(dx * dx + dy * dy));
        }
        double g = 0.0;
        m = grid_query(&gg, gpos, xi, yi, H * H, -1, &buf, &cap);
        for (int t = 0; t < m; t++) {
            int k = buf[t];
            double dx = xi - gpos[2 * k], dy = yi - gpos[2 * k + 1];
            g += orc_W_cb(p, sqrt(dx * dx + dy * dy));
        }
        sf[i] = f;
        sg[i] = g;
    }
    free(buf);
    grid_free(&gf);
    grid_free(&gg);
}

void orc_density(const orc_params* p, int n, const double* pos, int ng, const double* gpos,
                 double* rho, double* P) {
    double H = 2.0 * p->h;
    grid_t gf, gg;
    grid_build(&gf, n, pos, H);
    grid_build(&gg, ng, gpos, H);
    int cap = 64;
    int* buf = (int*)malloc(sizeof(int) * (size_t)cap);
    for (int i = 0; i < n; i++) {
        double xi = pos[2 * i], yi = pos[2 * i + 1];
        double sf = orc_W_cb(p, 0.0); /* self term first */
        int m = grid_query(&gf, pos, xi, yi, H * H, i, &buf, &cap);
        for (int t = 0; t < m; t++) {
            int j = buf[t];
            double dx = xi - pos[2 * j], dy = yi - pos[2 * j + 1];
            sf += orc_W_cb(p, sqrt(dx * dx + dy * dy));
        }
        double sg = 0.0;
        m = grid_query(&gg, gpos, xi, yi, H * H, -1, &buf, &cap);
        for (int t = 0; t < m; t++) {
            int g = buf[t];
            double dx = xi - gpos[2 * g], dy = yi - gpos[2 * g + 1];
            sg += orc_W_cb(p, sqrt(dx * dx + dy * dy));
        }
        rho[i] = p->mass * (sf + p->gamma1 * sg);
        P[i] = p->k * (rho[i] - p->rho0);                                   /* Eq. EOS */
        if (p->clamp_negative_pressure != 0.0 && P[i] < 0.0) P[i] = 0.0;
    }
    free(buf);
    grid_free(&gf);
    grid_free(&gg);
}

/* ------------------------------------------------------------------------------------ */
/* Steps 5-8: forces and accelerations.                                                    */
/* ------------------------------------------------------------------------------------ */
void orc_forces(const orc_params* p, int n, const double* pos, const double* vel,
                const double* rho, const double* P, int ng, const double* gpos,
                const double* gvel, const double* body, double* acc, double* Fb, double* Tb) {
    double h = p->h, H = 2.0 * h, m = p->mass;
    grid_t gf, gg;
    grid_build(&gf, n, pos, H);
    grid_build(&gg, ng, gpos, h);
    int cap = 64;
    int* buf = (int*)malloc(sizeof(int) * (size_t)cap);
    /* reaction force on each ghost:  F^{f2g}_{g<-i} = -F^{g2f}_{i<-g} */
    double* Fg = (double*)calloc((size_t)(ng > 0 ? ng : 1) * 2, sizeof(double));
    for (int i = 0; i < n; i++) {
        double xi = pos[2 * i], yi = pos[2 * i + 1], vxi = vel[2 * i], vyi = vel[2 * i + 1];
        double Fpx = 0, Fpy = 0, Fvx = 0, Fvy = 0;
        int M = grid_query(&gf, pos, xi, yi, H * H, i, &buf, &cap);
        for (int t = 0; t < M; t++) {
            int j = buf[t];
            double rx = xi - pos[2 * j], ry = yi - pos[2 * j + 1];
            double r = sqrt(rx * rx + ry * ry);
            double gx, gy;
            grad(orc_dW_cb(p, r), rx, ry, r, &gx, &gy);
            /* Eq. momentum: m_i sum_j m_j (P_i/rho_i^2 + P_j/rho_j^2) grad W */
            double cp = m * m * (P[i] / (rho[i] * rho[i]) + P[j] / (rho[j] * rho[j]));
            Fpx += cp * gx;
            Fpy += cp * gy;
            /* Eq. viscous: m_i sum_j m_j 2 alpha h/(rho_i+rho_j)
             *                          (rdot_ij . r_ij)/(|r_ij|^2 + eps h^2) grad W */
            double vr = (vxi - vel[2 * j]) * rx + (vyi - vel[2 * j + 1]) * ry;
            double cv = m * m * (2.0 * p->alpha * h / (rho[i] + rho[j])) * vr / (r * r + p->eps * h * h);
            Fvx += cv * gx;
            Fvy += cv * gy;
        }
        /* wall: spiky kernel, support h */
        double Gx = 0, Gy = 0;
        M = grid_query(&gg, gpos, xi, yi, h * h, -1, &buf, &cap);
        for (int t = 0; t < M; t++) {
            int g = buf[t];
            double rx = xi - gpos[2 * g], ry = yi - gpos[2 * g + 1];
            double r = sqrt(rx * rx + ry * ry);
            double gx, gy;
            grad(orc_dW_s3(p, r), rx, ry, r, &gx, &gy);
            double m_g = m, rho_g = rho[i]; /* ghosts inherit the fluid's properties */
            /* Eq. pressure_b2f with the wall sign of reading A4 */
            double cp = p->ghost_pressure_sign * 2.0 * m * m_g * P[i] / (rho[i] * rho[i]);
            /* Eq. viscous_b2f */
            double vr = (vxi - gvel[2 * g]) * rx + (vyi - gvel[2 * g + 1]) * ry;
            double cv = m * m_g * (2.0 * p->beta / (rho[i] + rho_g)) * (vr < 0.0 ? vr : 0.0) /
                        (r * r + p->eps * h * h);
            double Gix = (cp + cv) * gx, Giy = (cp + cv) * gy;
            Gx += Gix;
            Gy += Giy;
            Fg[2 * g] -= Gix;
            Fg[2 * g + 1] -= Giy;
        }
        /* Algorithm 1 l.8: a_i = m^-1 (-F^p + F^v + F^ext + F^g2f) */
        acc[2 * i] = (-Fpx + Fvx + Gx) / m + p->gx;
        acc[2 * i + 1] = (-Fpy + Fvy + Gy) / m + p->gy;
    }
    /* Eq. tankdynamics: F = sum_g sum_i F^{f2g}; T = sum_g (r_g - r) x sum_i F^{f2g} */
    double fx = 0, fy = 0, T = 0;
    for (int g = 0; g < ng; g++) {
        fx += Fg[2 * g];
        fy += Fg[2 * g + 1];
        double ax = gpos[2 * g] - body[0], ay = gpos[2 * g + 1] - body[1];
        T += ax * Fg[2 * g + 1] - ay * Fg[2 * g];
    }
    Fb[0] = fx;
    Fb[1] = fy;
    *Tb = T;
    free(Fg);
    free(buf);
    grid_free(&gf);
    grid_free(&gg);
}

/* ------------------------------------------------------------------------------------ */
/* One substep: Algorithm 1 + symplectic Euler kick-then-drift.         */
/* ------------------------------------------------------------------------------------ */
int orc_step(const orc_params* p, int n, double* pos, double* vel, int ng, const double* gB,
             double* body, const double* u, double damping, int pin_body, double* rho_out) {
    size_t nn = (size_t)(n > 0 ? n : 1), gg = (size_t)(ng > 0 ? ng : 1);
    double* gpos = (double*)malloc(sizeof(double) * 2 * gg);
    double* gvel = (double*)malloc(sizeof(double) * 2 * gg);
    double* rho = (double*)malloc(sizeof(double) * nn);
    double* P = (double*)malloc(sizeof(double) * nn);
    double* acc = (double*)malloc(sizeof(double) * 2 * nn);
    double Fb[2], Tb;
    orc_ghosts(ng, gB, body, gpos, gvel);                                  /* l.1-3 */
    orc_density(p, n, pos, ng, gpos, rho, P);                              /* l.5-6 */
    orc_forces(p, n, pos, vel, rho, P, ng, gpos, gvel, body, acc, Fb, &Tb); /* l.7-9 */
    double dt = p->dt;
    for (int i = 0; i < n; i++) {                                          /* kick, drift */
        vel[2 * i] += dt * acc[2 * i];
        vel[2 * i + 1] += dt * acc[2 * i + 1];
        pos[2 * i] += dt * vel[2 * i];
        pos[2 * i + 1] += dt * vel[2 * i + 1];
        vel[2 * i] *= damping;
        vel[2 * i + 1] *= damping;
    }
    if (!pin_body) {                                                       /* l.10 */
        double ax = (Fb[0] + u[0]) / p->m_body, ay = (Fb[1] + u[1]) / p->m_body;
        double ath = (Tb + u[2]) / p->J_body;
        body[3] += dt * ax;
        body[4] += dt * ay;
        body[5] += dt * ath;
        body[0] += dt * body[3];
        body[1] += dt * body[4];
        body[2] += dt * body[5];
    }
    if (rho_out) memcpy(rho_out, rho, sizeof(double) * (size_t)n);
    int st = 0;
    for (int i = 0; i < 2 * n && st == 0; i++) {
        if (!isfinite(pos[i]) || !isfinite(vel[i])) st = 1;
        else if (fabs(pos[i]) > 1e9 || fabs(vel[i]) > 1e9) st = 2;
    }
    for (int i = 0; i < 6 && st == 0; i++) {
        if (!isfinite(body[i])) st = 1;
        else if (fabs(body[i]) > 1e9) st = 2;
    }
    free(gpos);
    free(gvel);
    free(rho);
    free(P);
    free(acc);
    return st;
}

int orc_rollout(const orc_params* p, int n, double* pos, double* vel, int ng, const double* gB,
                double* body, int K, int n_sub, const double* u_seq, const double* theta_ref,
                double Kp, double Kd, double* y_out, double* u_applied, int64_t* bad_step) {
    *bad_step = -1;
    for (int k = 0; k < K; k++) {
        double u[3] = {u_seq[3 * k], u_seq[3 * k + 1], u_seq[3 * k + 2]};
        for (int c = 0; c < 6; c++) y_out[6 * k + c] = body[c]; /* y_k = y(k T_s), before u_k */
        if (theta_ref) u[2] = Kp * (theta_ref[k] - body[2]) - Kd * body[5];
        if (u_applied)
            for (int c = 0; c < 3; c++) u_applied[3 * k + c] = u[c];
        for (int s = 0; s < n_sub; s++) { /* ZOH over [k T_s, (k+1) T_s) */
            int st = orc_step(p, n, pos, vel, ng, gB, body, u, 1.0, 0, NULL);
            if (st) {
                *bad_step = (int64_t)k * n_sub + s;
                return st;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* float32 parity predicates (reading A19): IEEE single ops, -ffp-contract=off.            */
/* ------------------------------------------------------------------------------------ */
void orc_cells_f32(int n, const float* pos, float ox, float oy, float inv, int32_t* cells) {
    for (int i = 0; i < n; i++) {
        float tx = pos[2 * i] - ox;
        float ty = pos[2 * i + 1] - oy;
        tx = tx * inv;
        ty = ty * inv;
        cells[2 * i] = (int32_t)floorf(tx);
        cells[2 * i + 1] = (int32_t)floorf(ty);
    }
}

int64_t orc_neighbours_f32(int n, const float* pos, float H2, int64_t* off, int32_t* idx,
                           int64_t cap) {
    int64_t tot = 0;
    off[0] = 0;
    for (int i = 0; i < n; i++) {
        for (int j = 0; j < n; j++) {
            if (j == i) continue;
            float dx = pos[2 * i] - pos[2 * j];
            float dy = pos[2 * i + 1] - pos[2 * j + 1];
            float a = dx * dx;
            float b = dy * dy;
            float d2 = a + b;
            if (d2 < H2) {
                if (tot < cap) idx[tot] = j;
                tot++;
            }
        }
        off[i + 1] = tot;
    }
    return tot <= cap ? tot : -1;
}

int64_t orc_ghost_neighbours_f32(int n, const float* pos, int ng, const float* gpos, float R2,
                                 int64_t* off, int32_t* idx, int64_t cap) {
    int64_t tot = 0;
    off[0] = 0;
    for (int i = 0; i < n; i++) {
        for (int g = 0; g < ng; g++) {
            float dx = pos[2 * i] - gpos[2 * g];
            float dy = pos[2 * i + 1] - gpos[2 * g + 1];
            float a = dx * dx;
            float b = dy * dy;
            float d2 = a + b;
            if (d2 < R2) {
                if (tot < cap) idx[tot] = g;
                tot++;
            }
        }
        off[i + 1] = tot;
    }
    return tot <= cap ? tot : -1;
}

/* ---- linearization (P:259 item 2; SPEC linearization module) ----
 * Continuous-time state-transition function f of Sigma (Eq. NLmodel) with the state
 * laid out as x = [pos (n x 2, canonical id order), vel (n x 2), r_x, r_y, theta, rd_x, rd_y,
 * thd], n_x = 4n + 6, and u = (u_x, u_y, tau):
 *   d pos_i / dt = vel_i,  d vel_i / dt = a_i (Algorithm 1 l.1-8),
 *   d r / dt = rd,  d rd / dt = (F_b + u_xy) / m_B,  d theta / dt = thd,
 *   d thd / dt = (T_b + tau) / J   (Eq. tankdynamics).               */
void orc_deriv(const orc_params* p, int n, const double* x, int ng, const double* gB,
               const double* u, double* xdot) {
    size_t nn = (size_t)(n > 0 ? n : 1), gg = (size_t)(ng > 0 ? ng : 1);
    const double* pos = x;
    const double* vel = x + 2 * (size_t)n;
    const double* body = x + 4 * (size_t)n;
    double* gpos = (double*)malloc(sizeof(double) * 2 * gg);
    double* gvel = (double*)malloc(sizeof(double) * 2 * gg);
    double* rho = (double*)malloc(sizeof(double) * nn);
    double* P = (double*)malloc(sizeof(double) * nn);
    double* acc = (double*)malloc(sizeof(double) * 2 * nn);
    double Fb[2], Tb;
    orc_ghosts(ng, gB, body, gpos, gvel);                                  /* l.1-3 */
    orc_density(p, n, pos, ng, gpos, rho, P);                              /* l.5-6 */
    orc_forces(p, n, pos, vel, rho, P, ng, gpos, gvel, body, acc, Fb, &Tb); /* l.7-9 */
    for (int i = 0; i < 2 * n; i++) {
        xdot[i] = vel[i];
        xdot[2 * (size_t)n + i] = acc[i];
    }
    double* bd = xdot + 4 * (size_t)n;
    bd[0] = body[3];
    bd[1] = body[4];
    bd[2] = body[5];
    bd[3] = (Fb[0] + u[0]) / p->m_body;
    bd[4] = (Fb[1] + u[1]) / p->m_body;
    bd[5] = (Tb + u[2]) / p->J_body;
    free(gpos);
    free(gvel);
    free(rho);
    free(P);
    free(acc);
}

/* Central finite-difference Jacobian of f (the definition of the derivative, written out):
 * column j of A = (f(x + e_j h_j, u) - f(x - e_j h_j, u)) / (2 h_j), h_j = h_rel max(1, |x_j|);
 * B likewise for u.  A is n_x x n_x and B n_x x 3, row-major.  Truncation error O(h^2 f^(3)),
 * rounding O(eps |f| / h). */
void orc_jacobian_fd(const orc_params* p, int n, const double* x, int ng, const double* gB,
                     const double* u, double h_rel, double* A, double* B) {
    const int nx = 4 * n + 6;
    double* xp = (double*)malloc(sizeof(double) * (size_t)nx);
    double* fp = (double*)malloc(sizeof(double) * (size_t)nx);
    double* fm = (double*)malloc(sizeof(double) * (size_t)nx);
    double up[3], um[3];
    for (int j = 0; j < nx + 3; j++) {
        memcpy(xp, x, sizeof(double) * (size_t)nx);
        for (int c = 0; c < 3; c++) up[c] = um[c] = u[c];
        double hj;
        if (j < nx) {
            hj = h_rel * fmax(1.0, fabs(x[j]));
            xp[j] = x[j] + hj;
            orc_deriv(p, n, xp, ng, gB, u, fp);
            xp[j] = x[j] - hj;
            orc_deriv(p, n, xp, ng, gB, u, fm);
        } else {
            const int c = j - nx;
            hj = h_rel * fmax(1.0, fabs(u[c]));
            up[c] = u[c] + hj;
            um[c] = u[c] - hj;
            orc_deriv(p, n, x, ng, gB, up, fp);
            orc_deriv(p, n, x, ng, gB, um, fm);
        }
        for (int r = 0; r < nx; r++) {
            const double d = (fp[r] - fm[r]) / (2.0 * hj);
            if (j < nx) A[(size_t)r * nx + j] = d;
            else B[(size_t)r * 3 + (j - nx)] = d;
        }
    }
    free(xp);
    free(fp);
    free(fm);
}
