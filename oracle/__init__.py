"""ctypes shim over the float64 CPU oracle (oracle/orc.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs are the only callers.  The product package
(paper_2604_12505_b200) never imports this module, and this module never imports it.

parity status per function:
  W_cb, W_s3, dW_*      pinned (normalisation, closed forms, finite differences)
  neighbours*           pinned (brute force vs cell list; float32 predicate vs numpy)
  ghosts                pinned (rigidity, rotation special cases, golden G2)
  density               pinned (isolated particle, square-lattice sum, golden G1/G2)
  density_parts /
  estimate_gamma1       pinned (completed-lattice identity gamma1 = 1, ghost-doubling halves
                        it, density consistency, Table 2's gamma1 = 0.5 on the C1 wall layer)
  forces / step         pinned (golden G1/G2, momentum + angular momentum balance,
                        rigid-only closed form, hydrostatic identity, sign tests)
  rollout               pinned (PD gains, ZOH, sampling order vs closed forms)
  coupled trajectories beyond the invariants: parity unpinned (the paper prints no numbers)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liborc.so")
_SRC = os.path.join(_HERE, "orc.c")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle/orc.c -> oracle/liborc.so with gcc (no intrinsics, no contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "orc.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO + ".tmp", _SRC, "-lm"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


class Params(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "rho0", "k", "alpha", "beta", "gamma1", "eps", "h", "mass", "w_cb_const",
        "ghost_pressure_sign", "gx", "gy", "m_body", "J_body", "R", "dt", "clamp_negative_pressure")]


_lib = None
_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_F = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_I64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_I32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER(Params)
        for nm in ("orc_W_cb", "orc_dW_cb", "orc_W_s3", "orc_dW_s3"):
            getattr(L, nm).argtypes = [P, C.c_double]
            getattr(L, nm).restype = C.c_double
        L.orc_neighbours.argtypes = [P, C.c_int, _D, C.c_int, _I64, _I32, C.c_int64]
        L.orc_neighbours.restype = C.c_int64
        L.orc_ghosts.argtypes = [C.c_int, _D, _D, _D, _D]
        L.orc_density.argtypes = [P, C.c_int, _D, C.c_int, _D, _D, _D]
        L.orc_density_parts.argtypes = [P, C.c_int, _D, C.c_int, _D, _D, _D]
        L.orc_forces.argtypes = [P, C.c_int, _D, _D, _D, _D, C.c_int, _D, _D, _D, _D, _D,
                                 C.POINTER(C.c_double)]
        L.orc_step.argtypes = [P, C.c_int, _D, _D, C.c_int, _D, _D, _D, C.c_double, C.c_int,
                               C.c_void_p]
        L.orc_step.restype = C.c_int
        L.orc_rollout.argtypes = [P, C.c_int, _D, _D, C.c_int, _D, _D, C.c_int, C.c_int, _D,
                                  C.c_void_p, C.c_double, C.c_double, _D, C.c_void_p,
                                  C.POINTER(C.c_int64)]
        L.orc_rollout.restype = C.c_int
        L.orc_deriv.argtypes = [P, C.c_int, _D, C.c_int, _D, _D, _D]
        L.orc_jacobian_fd.argtypes = [P, C.c_int, _D, C.c_int, _D, _D, C.c_double, _D, _D]
        L.orc_cells_f32.argtypes = [C.c_int, _F, C.c_float, C.c_float, C.c_float, _I32]
        L.orc_neighbours_f32.argtypes = [C.c_int, _F, C.c_float, _I64, _I32, C.c_int64]
        L.orc_neighbours_f32.restype = C.c_int64
        L.orc_ghost_neighbours_f32.argtypes = [C.c_int, _F, C.c_int, _F, C.c_float, _I64, _I32,
                                               C.c_int64]
        L.orc_ghost_neighbours_f32.restype = C.c_int64
        _lib = L
    return _lib


def params(sp) -> Params:
    """orc params from a sph_inputs.SimParams (plain data)."""
    return Params(sp.rho0, sp.k, sp.alpha, sp.beta, sp.gamma1, sp.eps, sp.h, sp.mass,
                  sp.w_cb_const, sp.ghost_pressure_sign, sp.gx, sp.gy, sp.m_body, sp.J_body,
                  sp.R, sp.dt, float(getattr(sp, "clamp_negative_pressure", 0.0)))


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def W_cb(sp, r):
    return lib().orc_W_cb(C.byref(params(sp)), float(r))


def dW_cb(sp, r):
    return lib().orc_dW_cb(C.byref(params(sp)), float(r))


def W_s3(sp, r):
    return lib().orc_W_s3(C.byref(params(sp)), float(r))


def dW_s3(sp, r):
    return lib().orc_dW_s3(C.byref(params(sp)), float(r))


def _csr(fn, n, *args, cap=None):
    cap = cap or max(64, 16 * n)
    while True:
        off = np.zeros(n + 1, np.int64)
        idx = np.zeros(cap, np.int32)
        tot = fn(*args, off, idx, cap)
        if tot >= 0:
            return off, idx[:tot].copy()
        cap *= 4


def neighbours(sp, pos, use_cells=True):
    pos = _c(pos)
    n = pos.shape[0]
    return _csr(lambda o, i, c: lib().orc_neighbours(C.byref(params(sp)), n, pos, int(use_cells),
                                                     o, i, c), n)


def ghosts(ghost_b, body):
    gb = _c(ghost_b)
    ng = gb.shape[0]
    gp = np.zeros((ng, 2))
    gv = np.zeros((ng, 2))
    lib().orc_ghosts(ng, gb, _c(body), gp, gv)
    return gp, gv


def density(sp, pos, gpos):
    pos = _c(pos)
    gpos = _c(gpos).reshape(-1, 2)
    n = pos.shape[0]
    rho = np.zeros(n)
    P = np.zeros(n)
    lib().orc_density(C.byref(params(sp)), n, pos, gpos.shape[0], gpos, rho, P)
    return rho, P


def density_parts(sp, pos, gpos):
    """(sf, sg): the fluid (self included) and ghost kernel sums of Eq. density_update
    (P:180-182), rho_i = m (sf_i + gamma1 sg_i)."""
    pos = _c(pos)
    gpos = _c(gpos).reshape(-1, 2)
    n = pos.shape[0]
    sf = np.zeros(n)
    sg = np.zeros(n)
    lib().orc_density_parts(C.byref(params(sp)), n, pos, gpos.shape[0], gpos, sf, sg)
    return sf, sg


def estimate_gamma1(sp, pos, gpos, rho_target=None):
    """Analytic estimate of the wall correcting factor, Eq. gamma1:
        gamma1_i = (rho_i / m_i - sum_f W_i,f) / sum_g W_i,g
    with rho_i := rho_target (default rho0, the density the wall layer should have) and the
    printed denominator subscript i_b read as the ghost sum (reading G1).  Returns
    (gamma1_wall, gamma1_i, sf, sg): gamma1_i is NaN where no ghost is within 2h, and the single
    calibrated value gamma1_wall applies the same equation to the whole wall layer (the sums of
    its numerators and denominators over the particles with sg > 0: the gamma1 that gives the
    layer its target mass, reading G1)."""
    sf, sg = density_parts(sp, pos, gpos)
    rt = (sp.rho0 if rho_target is None else rho_target) / sp.mass
    w = sg > 0.0
    g = np.full(sf.shape, np.nan)
    g[w] = (rt - sf[w]) / sg[w]
    wall = float((rt - sf[w]).sum() / sg[w].sum()) if w.any() else float("nan")
    return wall, g, sf, sg


def forces(sp, pos, vel, rho, P, gpos, gvel, body):
    pos, vel = _c(pos), _c(vel)
    gpos, gvel = _c(gpos).reshape(-1, 2), _c(gvel).reshape(-1, 2)
    n = pos.shape[0]
    acc = np.zeros((n, 2))
    Fb = np.zeros(2)
    Tb = C.c_double(0.0)
    lib().orc_forces(C.byref(params(sp)), n, pos, vel, _c(rho), _c(P), gpos.shape[0], gpos, gvel,
                     _c(body), acc, Fb, C.byref(Tb))
    return acc, Fb, Tb.value


def state_vector(pos, vel, body):
    """x = [pos (n x 2), vel (n x 2), r_x, r_y, theta, rd_x, rd_y, thd] (orc_deriv layout)."""
    return np.concatenate([_c(pos).ravel(), _c(vel).ravel(), _c(body).ravel()])


def deriv(sp, x, ghost_b, u=(0.0, 0.0, 0.0)):
    """Continuous-time f(x, u) of Sigma in the state_vector layout."""
    x = _c(x)
    n = (x.shape[0] - 6) // 4
    gb = _c(ghost_b)
    out = np.zeros_like(x)
    lib().orc_deriv(C.byref(params(sp)), n, x, gb.shape[0], gb, _c(u), out)
    return out


def jacobian_fd(sp, x, ghost_b, u=(0.0, 0.0, 0.0), h_rel=1e-7):
    """Central-difference A = df/dx (n_x x n_x), B = df/du (n_x x 3) of f at (x, u).

    Default step 1e-7 (not SPEC's 1e-6): f has kinks (the one-sided wall viscosity
    min(v.r, 0), the kernels' higher derivatives at q = 1, 2 and r = h) and on C1 states a
    1e-6 stencil straddles one for a few entries (1e-4 relative change between h and 2h);
    at 1e-7 steps h and 2h agree to 2e-9 of max|A| and rounding stays ~eps |f| / h."""
    x = _c(x)
    nx = x.shape[0]
    n = (nx - 6) // 4
    gb = _c(ghost_b)
    A = np.zeros((nx, nx))
    B = np.zeros((nx, 3))
    lib().orc_jacobian_fd(C.byref(params(sp)), n, x, gb.shape[0], gb, _c(u), float(h_rel), A, B)
    return A, B


class State:
    """Mutable float64 oracle state of one rollout."""

    def __init__(self, sp, pos, vel, ghost_b, body=None):
        self.sp = sp
        self.p = params(sp)
        self.pos = _c(pos).copy()
        self.vel = _c(vel).copy()
        self.gb = _c(ghost_b).copy()
        self.body = np.zeros(6) if body is None else _c(body).copy()

    @classmethod
    def from_tank(cls, tank):
        return cls(tank.params, tank.pos, tank.vel, tank.ghost_b, tank.body)

    def step(self, u=(0.0, 0.0, 0.0), n=1, damping=1.0, pin_body=False, want_rho=False):
        u = _c(u)
        rho = np.zeros(self.pos.shape[0]) if want_rho else None
        for _ in range(n):
            st = lib().orc_step(C.byref(self.p), self.pos.shape[0], self.pos, self.vel,
                                self.gb.shape[0], self.gb, self.body, u, float(damping),
                                int(pin_body), rho.ctypes.data if want_rho else None)
            if st:
                raise FloatingPointError(f"oracle step failed with status {st}")
        return rho

    def rollout(self, u_seq, n_sub, theta_ref=None, Kp=0.0, Kd=0.0):
        u_seq = _c(u_seq).reshape(-1, 3)
        K = u_seq.shape[0]
        y = np.zeros((K, 6))
        ua = np.zeros((K, 3))
        th = _c(theta_ref) if theta_ref is not None else None
        bad = C.c_int64(-1)
        st = lib().orc_rollout(C.byref(self.p), self.pos.shape[0], self.pos, self.vel,
                               self.gb.shape[0], self.gb, self.body, K, int(n_sub), u_seq,
                               th.ctypes.data if th is not None else None, float(Kp), float(Kd),
                               y, ua.ctypes.data, C.byref(bad))
        if st:
            raise FloatingPointError(f"oracle rollout failed (status {st}) at substep {bad.value}")
        return y, ua


def settle(tank, seconds=4.0, rate=10.0):
    """Damped settle (reading A17): v <- v exp(-rate dt) after each step, body pinned at rest."""
    s = State.from_tank(tank)
    n = int(round(seconds / tank.params.dt))
    s.step(n=n, damping=float(np.exp(-rate * tank.params.dt)), pin_body=True)
    return s


# ---- float32 parity predicates (reading A19) -----------------------------------------
def cells_f32(pos32, ox, oy, inv):
    pos32 = _c(pos32, np.float32)
    n = pos32.shape[0]
    out = np.zeros((n, 2), np.int32)
    lib().orc_cells_f32(n, pos32, np.float32(ox), np.float32(oy), np.float32(inv), out)
    return out


def neighbours_f32(pos32, H2):
    pos32 = _c(pos32, np.float32)
    n = pos32.shape[0]
    return _csr(lambda o, i, c: lib().orc_neighbours_f32(n, pos32, np.float32(H2), o, i, c), n)


def ghost_neighbours_f32(pos32, gpos32, R2):
    pos32 = _c(pos32, np.float32)
    gpos32 = _c(gpos32, np.float32)
    n = pos32.shape[0]
    return _csr(lambda o, i, c: lib().orc_ghost_neighbours_f32(n, pos32, gpos32.shape[0], gpos32,
                                                               np.float32(R2), o, i, c), n)
