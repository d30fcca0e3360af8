"""Plain float64 oracle of the LPV surrogate (paper Sec. 4, and
Sec. 5.3).  TEST INFRASTRUCTURE ONLY (tests/, bench.py's cpu_baseline legs); the
product package never imports it and it imports nothing from the product.

Model (Eq. surrogate_form, Eq. LPVparametrization), benchmark dimensions of
P:438-440 (n_x = 4, n_u = 3, n_y = 3, n_p = 1, D = 0):
    p_k     = eta(x_k, u_k)                       FNN [x; u] -> 4 tanh -> 4 tanh -> n_p
    M(p_k)  = M_0 + p_k M_1,   M = [[A, B], [C, D]]
    x_{k+1} = A(p_k) x_k + B(p_k) u_k,   y^_k = C(p_k) x_k
Objective (Eqs. pem, surrogate_optimization P:303-310, regularization P:312-314):
    J + R = 1/N sum_k ||y_k - y^_k||^2 + sigma2/2 ||theta||^2 + sigmax/2 ||x0||^2
with several sequences: the mean of J over the sequences, one x0 per sequence (reading LPV3).
Fit measure: BFR (footnote of P:443).  Integrator augmentation: Eq. (28).

Parameter vector layout theta (n_theta = 137, SPEC's count; the paper prints 130, reading LPV1):
    A0 (4x4) B0 (4x3) C0 (3x4) A1 (4x4) B1 (4x3) C1 (3x4)   row-major, 80 values
    W1 (4x7) b1 (4) W2 (4x4) b2 (4) W3 (1x4) b3 (1)          57 values
The gradient is the definition of the derivative written out: central differences of the
objective (gradient_fd).

parity status: simulate / objective pinned (LTI collapse = scipy.signal.dlsim, constant
scheduling = dlsim of the frozen LTI, zero input); bfr pinned (closed forms); gradient_fd pinned
(step convergence); augment pinned (cumulative-sum identity).
"""
from __future__ import annotations

import numpy as np

NX, NU, NY, NPS, NH = 4, 3, 3, 1, 4
NZ = NX + NU
SIZES = [("A0", (NX, NX)), ("B0", (NX, NU)), ("C0", (NY, NX)),
         ("A1", (NX, NX)), ("B1", (NX, NU)), ("C1", (NY, NX)),
         ("W1", (NH, NZ)), ("b1", (NH,)), ("W2", (NH, NH)), ("b2", (NH,)),
         ("W3", (NPS, NH)), ("b3", (NPS,))]
N_THETA = sum(int(np.prod(s)) for _, s in SIZES)


def unpack(theta):
    """theta (flat, float64) -> dict of named arrays (views)."""
    theta = np.asarray(theta, np.float64)
    out, o = {}, 0
    for name, shp in SIZES:
        n = int(np.prod(shp))
        out[name] = theta[o:o + n].reshape(shp)
        o += n
    return out


def pack(parts):
    return np.concatenate([np.asarray(parts[name], np.float64).ravel() for name, _ in SIZES])


def eta(P, x, u):
    """Scheduling map: two tanh layers of 4, linear output."""
    z = np.concatenate([x, u])
    h1 = np.tanh(P["W1"] @ z + P["b1"])
    h2 = np.tanh(P["W2"] @ h1 + P["b2"])
    return P["W3"] @ h2 + P["b3"]


def simulate(theta, x0, u):
    """y^ [K, 3] and states x [K + 1, 4] of one sequence u [K, 3] (Eq. surrogate_form)."""
    P = unpack(theta)
    u = np.asarray(u, np.float64)
    K = u.shape[0]
    x = np.zeros((K + 1, NX))
    y = np.zeros((K, NY))
    x[0] = x0
    for k in range(K):
        p = eta(P, x[k], u[k])[0]
        A = P["A0"] + p * P["A1"]
        B = P["B0"] + p * P["B1"]
        C = P["C0"] + p * P["C1"]
        y[k] = C @ x[k]
        x[k + 1] = A @ x[k] + B @ u[k]
    return y, x


def objective(theta, x0s, us, ys, sigma2=1e-4, sigmax=1e-6):
    """J + R over S sequences: mean_s (1/K sum_k ||y - y^||^2) + sigma2/2 ||theta||^2
    + sigmax/2 sum_s ||x0_s||^2 (Eqs. pem, regularization)."""
    S = len(us)
    J = 0.0
    for s in range(S):
        yh, _ = simulate(theta, x0s[s], us[s])
        J += np.sum((np.asarray(ys[s], np.float64) - yh) ** 2) / us[s].shape[0]
    J /= S
    return J + 0.5 * sigma2 * np.sum(np.asarray(theta) ** 2) + 0.5 * sigmax * np.sum(np.asarray(x0s) ** 2)


def gradient_fd(theta, x0s, us, ys, sigma2=1e-4, sigmax=1e-6, h=1e-6):
    """Central differences of objective w.r.t. [theta, x0s.ravel()]."""
    theta = np.asarray(theta, np.float64)
    x0s = np.asarray(x0s, np.float64)
    v = np.concatenate([theta, x0s.ravel()])
    g = np.zeros_like(v)
    nt = theta.size

    def f(w):
        return objective(w[:nt], w[nt:].reshape(x0s.shape), us, ys, sigma2, sigmax)
    for i in range(v.size):
        e = np.zeros_like(v)
        e[i] = h * max(1.0, abs(v[i]))
        g[i] = (f(v + e) - f(v - e)) / (2.0 * e[i])
    return g


def bfr(y, yh):
    """Best fit rate per channel (footnote of P:443), in percent, not clipped."""
    y = np.asarray(y, np.float64)
    yh = np.asarray(yh, np.float64)
    num = np.sqrt(np.sum((y - yh) ** 2, axis=0))
    den = np.sqrt(np.sum((y - y.mean(0)) ** 2, axis=0))
    return (1.0 - num / den) * 100.0


def augment_outputs(yh, Ts, xe0=None):
    """Eq. (28) with D = 0: x^e_{k+1} = x^e_k + Ts C(p_k) x_k = x^e_k + Ts y^_k, so
    the position outputs are y^e_k = x^e_0 + Ts sum_{j<k} y^_j."""
    yh = np.asarray(yh, np.float64)
    xe = np.zeros_like(yh)
    acc = np.zeros(NY) if xe0 is None else np.asarray(xe0, np.float64).copy()
    for k in range(yh.shape[0]):
        xe[k] = acc
        acc = acc + Ts * yh[k]
    return xe
