"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no kernel, density, force or
integrator code).  It only produces *input data*: physical constants of the
paper's benchmark (Tables 1-2), the readings adopted where the paper is silent
(DESIGN.md "Readings"), initial particle lattices, the ghost ring in the body
frame, and input sequences u_k (manoeuvre profiles, excitation trains).

Citations: ``P:n`` = line n of the paper text (PAPER.md, arXiv 2604.12505).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict

import numpy as np

# --------------------------------------------------------------------------------------
# Physical constants (inputs).  Table 2, Table 1.
# --------------------------------------------------------------------------------------
RHO0 = 1017.0          # base density kg/m^2            (Table 2)
K_STIFF = 3.0          # stiffness k                    (Table 2)
ALPHA = 8.32e-4        # viscous factor                 (Table 2)
BETA = 4e-4            # boundary viscous factor        (Table 2)
GAMMA1 = 0.5           # correcting factor              (Table 2)
EPS = 0.01             # epsilon "~0.01"                (reading A9)
H_PAPER = 9.42e-3      # smoothing length h m           (Table 2)
D_PAPER = 6.0e-3       # "fuel particle length" m       (Table 2)
R_TANK = 0.2           # tank inner wall radius m       (Table 1)
M_BODY = 1010.71       # satellite mass kg              (Table 1)
J_BODY = 133.84        # satellite inertia kg m^2       (Table 1)
N_GHOST_PAPER = 236    # ghost particles                (Table 2)
N_FLUID_PAPER = 666    # fluid particles                (Table 2)
DT_PAPER = 1e-3        # fast step s
TS_PAPER = 0.05        # slow (sample/control) step s
PD_OMEGA = 0.2 * math.pi   # closed-loop bandwidth 0.1 Hz
PD_XI = 0.7                # damping ratio

# Reading A1: the printed cubic constant 15/(14 pi) integrates to 3, the
# normalised one (the paper asserts normalisation) is 5/(14 pi).
W_CB_CONST_NORMALISED = 5.0 / (14.0 * math.pi)
W_CB_CONST_PRINTED = 15.0 / (14.0 * math.pi)


@dataclass
class SimParams:
    """Every scalar the step needs.  Plain data; both sides receive the same values."""
    rho0: float = RHO0
    k: float = K_STIFF
    alpha: float = ALPHA
    beta: float = BETA
    gamma1: float = GAMMA1
    eps: float = EPS
    h: float = H_PAPER
    spacing: float = math.sqrt(3.0) * D_PAPER   # reading R1 (A2): lattice spacing s
    mass: float = RHO0 * 3.0 * D_PAPER ** 2     # reading R1: m = rho0 s^2
    w_cb_const: float = W_CB_CONST_NORMALISED   # reading A1
    ghost_pressure_sign: float = -1.0           # reading A4 (repulsive)
    clamp_negative_pressure: float = 0.0        # 0: Eq. EOS as printed; 1: P = max(P, 0) (ablation)
    gx: float = 0.0                             # zero gravity
    gy: float = 0.0
    m_body: float = M_BODY
    J_body: float = J_BODY
    R: float = R_TANK
    dt: float = DT_PAPER
    n_sub: int = 50                              # T_s / dt
    Kp: float = J_BODY * PD_OMEGA ** 2           # K = [J w^2, 2 xi J w]
    Kd: float = 2.0 * PD_XI * J_BODY * PD_OMEGA
    ell: float = 1.0

    def as_dict(self):
        return asdict(self)


def preset(ell: float = 1.0, **over) -> SimParams:
    """Refinement family of SURVEY 8(d): s = sqrt(3)*6mm/ell, h = 9.42mm/ell, dt = 1ms/ell."""
    s = math.sqrt(3.0) * D_PAPER / ell
    p = SimParams(h=H_PAPER / ell, spacing=s, mass=RHO0 * s * s, dt=DT_PAPER / ell,
                  n_sub=int(round(TS_PAPER / (DT_PAPER / ell))), ell=ell)
    for key, val in over.items():
        if not hasattr(p, key):
            raise KeyError(key)
        setattr(p, key, val)
    return p


# --------------------------------------------------------------------------------------
# Tank geometry (inputs): fluid lattice and ghost ring in the body frame.
# --------------------------------------------------------------------------------------
def ghost_ring(n_ghost: int, R: float = R_TANK) -> np.ndarray:
    """Body-frame ghost positions: n_g points uniformly on the wall circle."""
    j = np.arange(n_ghost, dtype=np.float64)
    phi = 2.0 * np.pi * j / n_ghost
    return np.stack([R * np.cos(phi), R * np.sin(phi)], axis=1)


def _segment_level(fill: float, R: float) -> float:
    """y_f such that the circular segment {y <= y_f} of the disk has area fill*pi*R^2 (bisection)."""
    target = fill * math.pi * R * R

    def area(y):
        y = max(-R, min(R, y))
        return R * R * math.acos(-y / R) + y * math.sqrt(max(R * R - y * y, 0.0))

    lo, hi = -R, R
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if area(mid) < target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def fluid_lattice(spacing: float, R: float = R_TANK, fill: float | None = 0.5,
                  n_first: int | None = None, jitter: float = 0.0, seed: int = 0) -> np.ndarray:
    """Square lattice sites (i s, j s) with |p| <= R - s/2, below the fill level y_f.

    Canonical particle ID = lexicographic (y, x) order.  ``n_first`` keeps the first n
    sites in that order with no fill level (the paper's 666-particle tank).
    ``jitter`` is a standard deviation in units of s, drawn from Philox(seed).
    """
    n = int(math.ceil(R / spacing)) + 1
    ii = np.arange(-n, n + 1, dtype=np.float64)
    X, Y = np.meshgrid(ii * spacing, ii * spacing)
    X = X.ravel()
    Y = Y.ravel()
    inside = X * X + Y * Y <= (R - 0.5 * spacing) ** 2
    if n_first is None and fill is not None:
        inside &= Y <= _segment_level(fill, R) + 1e-12
    X, Y = X[inside], Y[inside]
    order = np.lexsort((X, Y))
    pts = np.stack([X[order], Y[order]], axis=1)
    if n_first is not None:
        pts = pts[:n_first]
    if jitter > 0.0:
        rng = np.random.Generator(np.random.Philox(seed))
        pts = pts + rng.normal(0.0, jitter * spacing, size=pts.shape)
    return pts


@dataclass
class Tank:
    params: SimParams
    pos: np.ndarray           # [N_f, 2] float64 (float32-representable when snapped)
    vel: np.ndarray           # [N_f, 2]
    ghost_b: np.ndarray       # [N_g, 2] body frame
    body: np.ndarray = field(default_factory=lambda: np.zeros(6))  # r_x r_y th rd_x rd_y thd

    @property
    def n_fluid(self):
        return self.pos.shape[0]

    @property
    def n_ghost(self):
        return self.ghost_b.shape[0]

    def snapped(self) -> "Tank":
        """Round particle state to float32 (shared-input protocol)."""
        return Tank(self.params, self.pos.astype(np.float32).astype(np.float64),
                    self.vel.astype(np.float32).astype(np.float64),
                    self.ghost_b.astype(np.float32).astype(np.float64), self.body.copy())

    def pv32(self) -> np.ndarray:
        return np.ascontiguousarray(np.concatenate([self.pos, self.vel], axis=1).astype(np.float32))


def make_tank(ell: float = 1.0, fill: float | None = 0.5, n_first: int | None = None,
              jitter: float = 0.0, seed: int = 0, **over) -> Tank:
    """Config presets of SURVEY 8(d): C1 = make_tank(1), C2 = make_tank(4), C4 = make_tank(42),
    P0 = make_tank(1, n_first=666)."""
    p = preset(ell, **over)
    pos = fluid_lattice(p.spacing, p.R, fill=fill, n_first=n_first, jitter=jitter, seed=seed)
    ng = int(round(N_GHOST_PAPER * ell))
    return Tank(p, pos, np.zeros_like(pos), ghost_ring(ng, p.R))


def moving_tank(ell: float = 1.0, seed: int = 1, jitter: float = 0.05, vel: float = 0.01,
                body=None, **over) -> Tank:
    """Jittered lattice with random velocities (an unsettled, fully active state: one-step and
    linearization parity), rigidly placed at the body pose ``body`` = (r_x, r_y, th, rd_x,
    rd_y, thd) when given; snapped to float32-representable values."""
    t = make_tank(ell, jitter=jitter, seed=seed, **over)
    t.vel = np.random.Generator(np.random.Philox(seed + 100)).normal(0, vel, t.pos.shape)
    if body is not None:
        th = body[2]
        c, s = math.cos(th), math.sin(th)
        p = t.pos.copy()
        t.pos = np.stack([c * p[:, 0] - s * p[:, 1] + body[0], s * p[:, 0] + c * p[:, 1] + body[1]], 1)
        t.body = np.asarray(body, np.float64)
    return t.snapped()


def random_spawn(ell: float = 1.0, seed: int = 0, fill: float | None = 0.5,
                 n_first: int | None = None, **over) -> Tank:
    """Random-spawn initial state of the paper's settling procedure ("fuel particles
    are spawned randomly distributed within the tank and allowed to evolve without external
    actuation until their velocities converge to zero"): as many particles as make_tank(ell,
    fill, n_first) places (so the fluid mass is the same), uniformly distributed (Philox(seed),
    rejection sampling) over the region the lattice occupies -- |p| <= R - s/2 and, with a fill
    level, y <= y_f; with ``n_first`` (the P0 tank) below the level of the last lattice row.
    At rest, body at the origin; snapped to float32."""
    t = make_tank(ell, fill=fill, n_first=n_first, **over)
    p = t.params
    n = t.n_fluid
    y_top = _segment_level(fill, p.R) if n_first is None and fill is not None else \
        float(t.pos[:, 1].max()) + 0.5 * p.spacing
    rng = np.random.Generator(np.random.Philox(seed))
    pts = np.zeros((0, 2))
    while pts.shape[0] < n:
        c = rng.uniform(-p.R, p.R, size=(4 * n, 2))
        ok = (np.hypot(c[:, 0], c[:, 1]) <= p.R - 0.5 * p.spacing) & (c[:, 1] <= y_top)
        pts = np.concatenate([pts, c[ok]])
    pos = pts[:n]
    return Tank(p, pos, np.zeros_like(pos), t.ghost_b).snapped()


def random_tank(n_fluid: int, n_ghost: int, seed: int, h: float = H_PAPER, R: float = 0.03,
                vel_scale: float = 0.02, **over) -> Tank:
    """Small random (non-lattice) tank for parity edge cases: uniform points in the disk."""
    rng = np.random.Generator(np.random.Philox(seed))
    rr = R * np.sqrt(rng.uniform(0.0, 0.97, size=n_fluid))
    ph = rng.uniform(0.0, 2 * np.pi, size=n_fluid)
    pos = np.stack([rr * np.cos(ph), rr * np.sin(ph)], axis=1)
    vel = rng.normal(0.0, vel_scale, size=pos.shape)
    p = preset(1.0, h=h, R=R, **over)
    return Tank(p, pos, vel, ghost_ring(n_ghost, R))


# --------------------------------------------------------------------------------------
# Input sequences u_k (sampled at T_s; ZOH between samples).
# --------------------------------------------------------------------------------------
def profile(pid: int, K: int, Ts: float = TS_PAPER, rng: np.random.Generator | None = None):
    """Manoeuvre profiles 1 and 2 (magnitudes from SPEC defaults).

    Returns (u[K,3], theta_ref[K]).  With ``rng`` the amplitudes are scaled by U[0.5,1.5],
    pulse starts shifted by U[-1,1] s and the theta_ref step drawn from U[0.05,0.15] rad
    (SURVEY 8(d), config C5).
    """
    t = np.arange(K, dtype=np.float64) * Ts
    u = np.zeros((K, 3))
    th = np.zeros(K)
    a = (lambda: rng.uniform(0.5, 1.5)) if rng is not None else (lambda: 1.0)
    sh = (lambda: rng.uniform(-1.0, 1.0)) if rng is not None else (lambda: 0.0)
    if pid == 1:
        u[:, 0] = 5.0 * a()                                   # constant x thrust
        t_step = 5.0 + sh()
        th[t >= t_step] = rng.uniform(0.05, 0.15) if rng is not None else 0.1
        t0 = 15.0 + sh()
        u[(t >= t0) & (t < t0 + 0.5), 1] = 10.0 * a()        # y disturbance pulse
    elif pid == 2:
        amp = 10.0 * a()
        t0 = 2.0 + sh()
        t1 = 12.0 + sh()
        on = (t >= t0) & (t < t0 + 1.0)
        off = (t >= t1) & (t < t1 + 1.0)
        u[on, 0] = amp
        u[on, 1] = amp
        u[off, 0] = -amp
        u[off, 1] = -amp
    else:
        raise ValueError(pid)
    return u, th


def excitation(seed: int, K: int = 2200, Ts: float = TS_PAPER, rms=(2.0, 2.0, 1.0),
               n_pulses: int = 4, pulse_width: float = 1.0) -> np.ndarray:
    """Open-loop identification input train: per channel a multisine on the
    0.05 Hz grid below 2 Hz with random phases plus pulses (SURVEY 8(d) C3 recipe)."""
    rng = np.random.Generator(np.random.Philox(seed))
    t = np.arange(K, dtype=np.float64) * Ts
    u = np.zeros((K, 3))
    nfreq = np.arange(1, 40)
    for c in range(3):
        ph = rng.uniform(0.0, 2 * np.pi, size=nfreq.size)
        ms = np.cos(2 * np.pi * 0.05 * nfreq[None, :] * t[:, None] + ph[None, :]).sum(axis=1)
        u[:, c] = ms * (rms[c] / math.sqrt(nfreq.size / 2.0))
        horizon = K * Ts
        for _ in range(n_pulses):
            t0 = rng.uniform(0.0, max(horizon - pulse_width, 0.0))
            sgn = 1.0 if rng.uniform() < 0.5 else -1.0
            u[(t >= t0) & (t < t0 + pulse_width), c] += sgn * 2.0 * rms[c]
    return u


def ensemble_inputs(global_ids, K: int, kind: str = "excitation"):
    """Inputs for rollouts with the given GLOBAL ids (independent of sharding / batch position).

    kind="excitation": C3 (open loop, seed 1000 + id).  kind="profiles": C5 (ids with
    id < n/2 get profile 1, others profile 2; randomised with seed 2000 + id) -> the caller
    passes ``n_total`` via ids' maximum.  Returns (u[B,K,3] float32, theta_ref[B,K] or None).
    """
    ids = list(global_ids)
    if kind == "excitation":
        u = np.stack([excitation(1000 + g, K=max(K, 1))[:K] for g in ids]).astype(np.float32)
        return u, None
    raise ValueError(kind)


def profile_inputs(global_ids, n_total: int, K: int):
    us, ths = [], []
    for g in global_ids:
        rng = np.random.Generator(np.random.Philox(2000 + g))
        u, th = profile(1 if g < n_total // 2 else 2, K, rng=rng)
        us.append(u)
        ths.append(th)
    return np.stack(us).astype(np.float32), np.stack(ths).astype(np.float32)
