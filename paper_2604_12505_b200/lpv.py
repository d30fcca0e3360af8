"""LPV surrogate identification on the GPU (paper Sec. 4, and Sec.
5.3): the consumer of the simulator's datasets.

Every evaluation of the model, the objective and its gradient runs in the CUDA kernel behind
``sph_lpv_eval`` (one launch per optimiser step for all restarts); Adam steps run in
``sph_lpv_adam``.  This module marshals arguments and runs the optimiser's control logic
(L-BFGS two-loop recursion and backtracking line search on the 137 + 4S parameters of each
restart, in lockstep over the restarts).

Model and parameter layout: include/sph.h (SPH_LPV_NTHETA); readings LPV1-LPV4 in DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from .binding import SphError, SPH_OK, lib

NX, NU, NY, NH, NZ = 4, 3, 3, 4, 7
NT = 137
LAYOUT = [("A0", (4, 4)), ("B0", (4, 3)), ("C0", (3, 4)), ("A1", (4, 4)), ("B1", (4, 3)),
          ("C1", (3, 4)), ("W1", (4, 7)), ("b1", (4,)), ("W2", (4, 4)), ("b2", (4,)),
          ("W3", (1, 4)), ("b3", (1,))]
OFF = {}
_o = 0
for _n, _s in LAYOUT:
    OFF[_n] = (_o, _s)
    _o += int(np.prod(_s))
assert _o == NT


def block(theta, name):
    o, s = OFF[name]
    return np.asarray(theta)[..., o:o + int(np.prod(s))].reshape(np.asarray(theta).shape[:-1] + s)


def normalise(us, ys, center=False):
    """Per-channel scaling of the training record ("scaled and normalized dataset", P:444;
    reading LPV4): divide by the RMS, no mean shift by default -- the model has no affine term
    and the velocity-level dynamics integrate the input, so a shifted input would add a ramp the
    model cannot represent (center=True: SPEC's standardisation).  Returns (u_n, y_n,
    (u_offset, u_scale, y_offset, y_scale)); physical = offset + scale * normalised."""
    U = np.concatenate(us, 0)
    Y = np.concatenate(ys, 0)
    um = U.mean(0) if center else np.zeros(U.shape[1])
    ym = Y.mean(0) if center else np.zeros(Y.shape[1])
    usd = np.sqrt(((U - um) ** 2).mean(0))
    ysd = np.sqrt(((Y - ym) ** 2).mean(0))
    usd[usd == 0] = 1.0
    ysd[ysd == 0] = 1.0
    un = [((u - um) / usd).astype(np.float32) for u in us]
    yn = [((y - ym) / ysd).astype(np.float32) for y in ys]
    return un, yn, (um, usd, ym, ysd)


def bfr(y, yh):
    """Best fit rate per channel (footnote of P:443), percent, not clipped."""
    y = np.asarray(y, np.float64)
    yh = np.asarray(yh, np.float64)
    return (1.0 - np.sqrt(((y - yh) ** 2).sum(0)) / np.sqrt(((y - y.mean(0)) ** 2).sum(0))) * 100.0


def augment_positions(yh, Ts, xe0=None):
    """Eq. (28), D = 0: x^e_{k+1} = x^e_k + Ts y^_k -> position outputs."""
    yh = np.asarray(yh, np.float64)
    c = np.cumsum(yh, 0) * Ts
    out = np.vstack([np.zeros((1, yh.shape[1])), c[:-1]])
    return out if xe0 is None else out + np.asarray(xe0, np.float64)


def init_params(R, S, seed, lti=None, m1_std=0.01):
    """Restart initialisations: M0 from the LTI fit (``lti``: theta with M0 set) or,
    without one, A0 = 0.9 I + N(0, 0.01) and B0, C0 ~ N(0, 0.1); M1 ~ N(0, m1_std) ("zero-mean
    normal", std reading LPV2); eta weights Xavier-uniform (Glorot), biases 0; x0 = 0."""
    rng = np.random.Generator(np.random.Philox(seed))
    P = np.zeros((R, NT + NX * S))
    for r in range(R):
        th = P[r, :NT]
        if lti is not None:
            th[:OFF["A1"][0]] = np.asarray(lti)[:OFF["A1"][0]]
        else:
            th[OFF["A0"][0]:OFF["B0"][0]] = (0.9 * np.eye(4) + rng.normal(0, 0.01, (4, 4))).ravel()
            th[OFF["B0"][0]:OFF["A1"][0]] = rng.normal(0, 0.1, 24)
        th[OFF["A1"][0]:OFF["W1"][0]] = rng.normal(0, m1_std, 40)
        for name, fan_in, fan_out in (("W1", 7, 4), ("W2", 4, 4), ("W3", 4, 1)):
            o, s = OFF[name]
            lim = math.sqrt(6.0 / (fan_in + fan_out))
            th[o:o + int(np.prod(s))] = rng.uniform(-lim, lim, int(np.prod(s)))
    return P


class LpvProblem:
    """R parameter sets (restarts) x S sequences of K samples, device resident.

    us, ys: lists of S arrays [K, 3] (already normalised; ys may be None for simulation only)."""

    def __init__(self, R, us, ys=None, sigma2=1e-4, sigmax=1e-6, device=0):
        import torch
        self.torch = torch
        self.L = lib()
        self.dev = torch.device("cuda", device)
        self.R, self.S, self.K = int(R), len(us), int(us[0].shape[0])
        self.n = NT + NX * self.S
        self.sigma2, self.sigmax = float(sigma2), float(sigmax)
        f32 = torch.float32
        self.u = torch.from_numpy(np.ascontiguousarray(np.stack(us), np.float32)).to(self.dev)
        self.y = None if ys is None else \
            torch.from_numpy(np.ascontiguousarray(np.stack(ys), np.float32)).to(self.dev)
        self.params = torch.zeros((self.R, self.n), dtype=torch.float64, device=self.dev)
        self.grad = torch.zeros_like(self.params)
        self.obj = torch.zeros(self.R, dtype=torch.float64, device=self.dev)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        nb = int(self.L.sph_lpv_scratch_bytes(self.R, self.S, self.K))
        if nb == 0:
            raise SphError("sph_lpv_scratch_bytes: bad sizes")
        self.scratch = torch.empty(nb, dtype=torch.uint8, device=self.dev)
        self.stream = torch.cuda.current_stream(self.dev)
        self.t = 0
        self.mask = None
        self.yhat = torch.empty((self.R, self.S, self.K, NY), dtype=f32, device=self.dev)

    def _chk(self, st, what):
        if st != SPH_OK:
            raise SphError(f"{what}: status {st}")

    def set_params(self, P):
        self.params.copy_(self.torch.from_numpy(np.ascontiguousarray(P, np.float64)))
        self.m.zero_()
        self.v.zero_()
        self.t = 0

    def set_mask(self, trainable):
        """trainable: bool [n] (None: all); frozen parameters keep their values under Adam."""
        self.mask = None if trainable is None else \
            self.torch.from_numpy(np.asarray(trainable, np.uint8)).to(self.dev)

    def eval(self, params=None, grad=True, yhat=False):
        """Objective [R] (and gradient [R, n]) at ``params`` (device tensor; default: current)."""
        p = self.params if params is None else params
        self._chk(self.L.sph_lpv_eval(
            self.R, self.S, self.K, p.data_ptr(), self.u.data_ptr(),
            None if self.y is None else self.y.data_ptr(), self.sigma2, self.sigmax,
            None if self.y is None else self.obj.data_ptr(),
            self.grad.data_ptr() if grad else None,
            self.yhat.data_ptr() if yhat else None,
            self.scratch.data_ptr(), self.scratch.numel(), C.c_void_p(self.stream.cuda_stream)),
            "sph_lpv_eval")
        return self.obj, (self.grad if grad else None)

    def adam(self, iters, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        """``iters`` Adam steps: one eval + one fused update launch each."""
        for _ in range(iters):
            self.eval()
            self.t += 1
            self._chk(self.L.sph_lpv_adam(
                self.R, self.n, self.params.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                self.v.data_ptr(), lr, beta1, beta2, eps, self.t,
                None if self.mask is None else self.mask.data_ptr(),
                C.c_void_p(self.stream.cuda_stream)), "sph_lpv_adam")

    def lbfgs(self, max_iter, memory=10, tol_grad=1e-9, ftol=2.2e-9, c1=1e-4, max_backtrack=30):
        """L-BFGS ("warm-start a ... L-BFGS scheme") over the restarts: two-loop recursion
        (memory 10, vectorised over the restarts) and Armijo backtracking.  The restarts do not
        wait for each other: every launch evaluates each restart's current trial point, and a
        restart whose trial is accepted proceeds to its next direction while another backtracks
        (each launch advances every restart by one trial).  A restart stops after max_iter
        accepted iterations, when its gradient norm falls below tol_grad, its relative decrease
        (f_k - f_k+1) / max(|f_k|, |f_k+1|, 1) falls to ftol (scipy's L-BFGS-B default;
        reading LPV6), or its line search fails.  Frozen parameters (mask) stay fixed.
        Returns the number of objective evaluations (launches x restarts)."""
        torch = self.torch
        mk = None if self.mask is None else self.mask.cpu().numpy().astype(bool)
        f, g = self.eval()
        x = self.params.cpu().numpy()
        f = f.cpu().numpy().copy()
        g = g.cpu().numpy().copy()
        if mk is not None:
            g[:, ~mk] = 0.0
        R, n, m = self.R, self.n, int(memory)
        ar = np.arange(R)
        Sh = np.zeros((R, m, n))
        Yh = np.zeros((R, m, n))
        rh = np.zeros((R, m))
        cnt = np.zeros(R, np.int64)
        head = np.zeros(R, np.int64)          # next slot of each restart's circular history
        active = np.linalg.norm(g, axis=1) > tol_grad
        iters = np.zeros(R, np.int64)
        n_eval = 1

        def directions(sel):
            """Two-loop recursion for the restarts in ``sel`` (bool [R]); others get 0."""
            q = -g
            al = np.zeros((R, m))
            for j in range(m):                                   # newest -> oldest
                idx = (head - 1 - j) % m
                v = j < cnt
                a = np.where(v, rh[ar, idx] * np.einsum("rn,rn->r", Sh[ar, idx], q), 0.0)
                q = q - a[:, None] * Yh[ar, idx]
                al[:, j] = a
            last = (head - 1) % m
            sy = np.einsum("rn,rn->r", Sh[ar, last], Yh[ar, last])
            yy = np.einsum("rn,rn->r", Yh[ar, last], Yh[ar, last])
            g1 = np.maximum(np.abs(g).sum(1), 1e-300)
            gam = np.where(cnt > 0, sy / np.where(yy > 0, yy, 1.0), np.minimum(1.0, 1.0 / g1))
            q = q * gam[:, None]
            for j in reversed(range(m)):                         # oldest -> newest
                idx = (head - 1 - j) % m
                v = j < cnt
                b = rh[ar, idx] * np.einsum("rn,rn->r", Yh[ar, idx], q)
                q = q + np.where(v, al[:, j] - b, 0.0)[:, None] * Sh[ar, idx]
            bad = sel & ((g * q).sum(1) >= 0)     # not a descent direction: restart memory
            if bad.any():
                cnt[bad] = 0
                q[bad] = -g[bad] * np.minimum(1.0, 1.0 / g1[bad])[:, None]
            return np.where(sel[:, None], q, 0.0)

        d = directions(active)
        slope = (g * d).sum(1)
        step = np.where(active, 1.0, 0.0)
        nbt = np.zeros(R, np.int64)
        while active.any():
            trial = np.where(active[:, None], x + step[:, None] * d, x)
            fo, go = self.eval(torch.from_numpy(trial).to(self.dev))
            n_eval += 1
            fo = fo.cpu().numpy()
            go = go.cpu().numpy()
            if mk is not None:
                go[:, ~mk] = 0.0
            ok = active & np.isfinite(fo) & (fo <= f + c1 * step * slope)
            # rejected trials backtrack; exhausted line searches stop their restart
            rej = active & ~ok
            nbt[rej] += 1
            step[rej] *= 0.5
            active &= ~(rej & (nbt >= max_backtrack))
            if ok.any():
                s_ = trial - x
                y_ = go - g
                sy = np.einsum("rn,rn->r", s_, y_)
                keep = ok & (sy > 1e-12 * np.linalg.norm(s_, axis=1) * np.linalg.norm(y_, axis=1))
                kk = np.flatnonzero(keep)
                Sh[kk, head[kk]] = s_[kk]
                Yh[kk, head[kk]] = y_[kk]
                rh[kk, head[kk]] = 1.0 / sy[kk]
                head[kk] = (head[kk] + 1) % m
                cnt[kk] = np.minimum(cnt[kk] + 1, m)
                stalled = ok & ((f - fo) <= ftol * np.maximum(np.maximum(np.abs(f), np.abs(fo)), 1.0))
                x[ok], f[ok], g[ok] = trial[ok], fo[ok], go[ok]
                iters[ok] += 1
                active &= ~stalled
                active &= ~(ok & (iters >= max_iter))
                active &= ~(ok & (np.linalg.norm(g, axis=1) <= tol_grad))
                nxt = ok & active
                if nxt.any():
                    dn = directions(nxt)
                    d[nxt] = dn[nxt]
                    slope[nxt] = (g[nxt] * d[nxt]).sum(1)
                    step[nxt] = 1.0
                    nbt[nxt] = 0
        self.params.copy_(torch.from_numpy(x))
        return n_eval

    def simulate(self, params=None):
        """y^ [R, S, K, 3] (normalised units) at ``params``."""
        self.eval(params, grad=False, yhat=True)
        return self.yhat


def arx_init(us, ys, device=0, slosh_pole=0.9):
    """LTI initial guess (reading LPV2; the paper uses MATLAB's ssest): least-squares ARX(1,1)
    fit y_{k+1} = Ay y_k + By u_k on the GPU (torch.linalg.lstsq, a library solve), the three
    measured outputs taken as the first three states; the fourth state starts decoupled with
    pole ``slosh_pole``.  Returns theta with M0 = (A0, B0, C0 = [I 0]) and the rest zero."""
    import torch
    dev = torch.device("cuda", device)
    X = torch.cat([torch.from_numpy(np.hstack([y[:-1], u[:-1]])) for u, y in zip(us, ys)]).to(dev, torch.float64)
    T = torch.cat([torch.from_numpy(np.asarray(y[1:], np.float64)) for y in ys]).to(dev)
    W = torch.linalg.lstsq(X, T).solution.cpu().numpy()        # [6, 3]: [Ay^T; By^T]
    th = np.zeros(NT)
    A0 = np.zeros((4, 4))
    A0[:3, :3] = W[:3].T
    A0[3, 3] = slosh_pole
    B0 = np.zeros((4, 3))
    B0[:3] = W[3:].T
    C0 = np.zeros((3, 4))
    C0[:, :3] = np.eye(3)
    for name, v in (("A0", A0), ("B0", B0), ("C0", C0)):
        o, sh = OFF[name]
        th[o:o + v.size] = v.ravel()
    return th


def identify(us, ys, restarts=8, adam_iters=2000, lbfgs_iters=6000, lti_iters=2000, seed=0,
             lr=1e-3, sigma2=1e-4, sigmax=1e-6, device=0, ftol=2.2e-9):
    """The identification procedure of P:441-446 on (normalised) sequences us, ys:
    1. LTI initialisation (reading LPV2): ARX(1,1) least squares (arx_init), then the M0 block
       (and x0) refined alone on the simulation error, Adam then L-BFGS (M1 = 0, eta frozen);
    2. ``restarts`` LPV restarts from that M0 with random M1 and Xavier eta: Adam then L-BFGS;
    3. the restart with the highest average training BFR.
    Returns dict(theta, x0, bfr_lti, bfr, bfr_all, n_evals)."""
    S = len(us)
    lti = LpvProblem(1, us, ys, sigma2, sigmax, device)
    P0 = np.zeros((1, NT + NX * S))
    P0[0, :NT] = arx_init(us, ys, device)
    for s_ in range(S):                      # x0: the first measured outputs
        P0[0, NT + NX * s_:NT + NX * s_ + 3] = np.asarray(ys[s_][0], np.float64)
    lti.set_params(P0)
    trainable = np.zeros(NT + NX * S, bool)
    trainable[:OFF["A1"][0]] = True
    trainable[NT:] = True
    lti.set_mask(trainable)
    lti.adam(lti_iters, lr=lr)
    n_ev = lti_iters + lti.lbfgs(lbfgs_iters // 2, ftol=ftol)
    th_lti = lti.params[0].cpu().numpy()
    yl = lti.simulate()[0].cpu().numpy()
    bfr_lti = float(np.mean([bfr(ys[s], yl[s]).mean() for s in range(S)]))
    prob = LpvProblem(restarts, us, ys, sigma2, sigmax, device)
    P = init_params(restarts, S, seed + 1, lti=th_lti)
    P[:, NT:] = th_lti[NT:]
    prob.set_params(P)
    prob.adam(adam_iters, lr=lr)
    n_ev += restarts * (adam_iters + prob.lbfgs(lbfgs_iters, ftol=ftol))
    yh = prob.simulate().cpu().numpy()
    fits = np.array([np.mean([bfr(ys[s], yh[r, s]).mean() for s in range(S)]) for r in range(restarts)])
    fits[~np.isfinite(fits)] = -np.inf
    best = int(np.argmax(fits))
    th = prob.params[best].cpu().numpy()
    return {"theta": th[:NT], "x0": th[NT:].reshape(S, NX), "bfr_lti": bfr_lti,
            "bfr": float(fits[best]), "bfr_all": fits.tolist(), "best": best, "n_evals": n_ev}
