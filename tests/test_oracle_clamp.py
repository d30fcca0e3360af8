"""Pins of the oracle's clamped-EOS ablation (SURVEY 8(b) clamp_negative_pressure; E1):
P = max(k (rho - rho0), 0).  A wall-free lattice at rest has rho <= rho0 everywhere (interior
0.99968 rho0 under reading R1, lower at its edges), so with the clamp every pressure vanishes
and the accelerations are exactly zero, while the literal EOS pulls the edges inward."""
import numpy as np

import oracle as O
import sph_inputs as si


def test_clamped_lattice_is_force_free():
    t = si.make_tank(1.0, clamp_negative_pressure=1.0)
    none = np.zeros((0, 2))
    rho, P = O.density(t.params, t.pos, none)
    assert rho.max() < t.params.rho0 and np.all(P == 0.0)
    acc, Fb, Tb = O.forces(t.params, t.pos, np.zeros_like(t.pos), rho, P, none, none, np.zeros(6))
    assert np.all(acc == 0.0) and np.all(Fb == 0.0) and Tb == 0.0
    t0 = si.make_tank(1.0)
    rho0, P0 = O.density(t0.params, t0.pos, none)
    assert np.array_equal(rho0, rho) and P0.min() < 0.0
    acc0, _, _ = O.forces(t0.params, t0.pos, np.zeros_like(t0.pos), rho0, P0, none, none, np.zeros(6))
    assert np.abs(acc0).max() > 0.0


def test_clamp_keeps_positive_pressures():
    t = si.moving_tank(1.0, seed=4, vel=0.0)
    gp, _ = O.ghosts(t.ghost_b, np.zeros(6))
    tc = si.moving_tank(1.0, seed=4, vel=0.0, clamp_negative_pressure=1.0)
    _, P = O.density(t.params, t.pos, gp)
    _, Pc = O.density(tc.params, tc.pos, gp)
    assert (P > 0).any() and (P < 0).any()
    assert np.array_equal(Pc[P > 0], P[P > 0]) and np.all(Pc[P <= 0] == 0.0)
