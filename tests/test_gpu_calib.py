"""SURVEY 8(f) f4 on the GPU: the gamma1 estimate (sph_gamma1_estimate, Eq. gamma1)
against the oracle's (tests/test_oracle_gamma1.py pins it), the paper's random-spawn settling
 on the device against the oracle's settle of the same spawn, and the readings'
ablations (literal ghost-pressure sign, printed cubic constant, R0 lattice; A1/A4/F4)
classified identically by both sides."""
import math
import os

import numpy as np
import pytest

import oracle as O
import sph_inputs as si

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ctx(t, B=1, **kw):
    from paper_2604_12505_b200 import SphContext
    return SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=B, **kw)


def _gamma1_case(t):
    ctx = _ctx(t)
    ctx.set_body_state(np.array([t.body]))
    wall, g, sums = ctx.gamma1_estimate(0)
    ctx.close()
    gp, _ = O.ghosts(t.ghost_b, t.body)
    wo, go, sf, sg = O.estimate_gamma1(t.params, t.pos, gp)
    sp = t.params
    unit = sp.w_cb_const / sp.h ** 2                       # sums are in units of C/h^2
    assert np.allclose(sums[:, 0], sf / unit, rtol=2e-6, atol=0)
    assert np.allclose(sums[:, 1], sg / unit, rtol=0, atol=2e-6 * np.abs(sf / unit).max())
    fin = np.isfinite(go)
    assert np.array_equal(np.isfinite(g), fin) and fin.sum() > 0
    rt = sp.rho0 / sp.mass / unit
    tol = 4e-6 * rt / (sg[fin] / unit)                     # float32 sums, cancellation in rt - sf
    assert np.all(np.abs(g[fin] - go[fin]) <= tol)
    assert abs(wall - wo) <= 2e-5 * abs(wo)
    return wall


def test_gamma1_estimate_rest_lattice():
    w = _gamma1_case(si.make_tank(1.0))
    assert 0.45 <= w <= 0.6                                # Table 2: gamma1 = 0.5


def test_gamma1_estimate_moving_rotated():
    _gamma1_case(si.moving_tank(1.0, seed=6, vel=0.0, body=[0.03, -0.02, 0.7, 0.0, 0.0, 0.0]))


def test_gamma1_estimate_settled_c2():
    snap = np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"].astype(np.float64)
    t = si.make_tank(4.0)
    _gamma1_case(si.Tank(t.params, snap[:, :2], snap[:, 2:], t.ghost_b).snapped())


def test_random_spawn_settle_matches_oracle():
    """random spawn, evolve without actuation until the velocities vanish (damped,
    reading A17, body pinned).  The trajectories are chaotic in the violent first phase, so the
    two sides are compared on what the settled state fixes: at rest, inside the wall, at the
    rest density, and with the same fluid centroid."""
    t = si.random_spawn(1.0, seed=11)
    sp = t.params
    n = int(round(3.0 / sp.dt))
    damp = math.exp(-10.0 * sp.dt)
    ctx = _ctx(t)
    ctx.settle(damp, n)
    st = ctx.get_status()[0]
    pv = ctx.get_particles(0).astype(np.float64)
    ctx.step(np.zeros((1, 3), np.float32), 1)
    _, rho = ctx.get_particles(0, with_rho=True)
    ctx.close()
    s = O.State.from_tank(t)
    s.step(n=n, damping=damp, pin_body=True)
    rho_o = s.step(n=1, want_rho=True, pin_body=True)
    assert st[0] == 0
    for pos, vel, r in ((pv[:, :2], pv[:, 2:], rho), (s.pos, s.vel, rho_o)):
        assert np.abs(vel).max() < 2e-3                     # converged to rest (from ~0.3 m/s)
        assert np.hypot(pos[:, 0], pos[:, 1]).max() < sp.R   # nothing tunnelled
        assert abs(np.median(r) / sp.rho0 - 1.0) < 2e-3
    assert np.abs(pv[:, :2].mean(0) - s.pos.mean(0)).max() < 2e-3 * sp.R


@pytest.mark.parametrize("reading", ["adopted", "literal_sign", "printed_constant", "R0"])
def test_reading_ablations_classified_alike(reading):
    """SURVEY F3/F4 probes: the P0 tank from its rest lattice, 3 s without actuation (body
    pinned).  Adopted readings keep every particle inside the wall on both sides; the literal
    ghost-pressure sign (attractive wall), the printed cubic constant and the R0 lattice let
    particles tunnel through it on both sides."""
    s0 = si.D_PAPER
    over = {"adopted": {}, "literal_sign": {"ghost_pressure_sign": 1.0},
            "printed_constant": {"w_cb_const": si.W_CB_CONST_PRINTED},
            "R0": {"spacing": s0, "mass": si.RHO0 * s0 * s0,
                   "w_cb_const": si.W_CB_CONST_PRINTED}}[reading]
    t = si.make_tank(1.0, n_first=666, **over).snapped()
    sp = t.params
    n = int(round(3.0 / sp.dt))
    ctx = _ctx(t)
    ctx.settle(1.0, n)
    st = ctx.get_status()[0]
    pv = ctx.get_particles(0).astype(np.float64)
    ctx.close()
    s = O.State.from_tank(t)
    s.step(n=n, pin_body=True)
    out_g = int((np.hypot(pv[:, 0], pv[:, 1]) > sp.R).sum())
    out_o = int((np.hypot(s.pos[:, 0], s.pos[:, 1]) > sp.R).sum())
    if reading == "adopted":
        assert st[0] == 0 and out_g == 0 and out_o == 0
    else:
        # the GPU side reports a particle that left its cell grid (status 3: tunnelled far
        # beyond the wall) and freezes the rollout; either way it tunnelled
        assert st[0] in (0, 3) and (st[0] == 3 or out_g > 0)
        assert out_o > 0
        if reading in ("literal_sign", "R0"):
            assert out_o > 0.2 * t.n_fluid


def test_settle_until_converges():
    """sph_settle_until ("until their velocities converge to zero"): a random spawn of the
    C1 tank settles below 2e-3 m/s in chunks of 250 substeps; an already converged state takes
    one chunk; the reported speed is the largest fluid speed of the returned state."""
    t = si.random_spawn(1.0, seed=12)
    sp = t.params
    damp = math.exp(-10.0 * sp.dt)
    ctx = _ctx(t)
    n, v = ctx.settle_until(damp, 2e-3, int(4.0 / sp.dt), 250)
    pv = ctx.get_particles(0).astype(np.float64)
    assert 0 < n < int(4.0 / sp.dt) and n % 250 == 0
    assert v[0] < 2e-3 and abs(np.hypot(pv[:, 2], pv[:, 3]).max() - v[0]) <= 1e-6
    n2, v2 = ctx.settle_until(damp, 1.0, 1000, 250)     # converged: one chunk, then the test
    assert n2 == 250 and v2[0] < v[0]
    ctx.close()
