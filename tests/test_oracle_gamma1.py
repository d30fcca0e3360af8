"""Pins of the oracle's gamma1 estimate (Eq. gamma1) against what
the geometry fixes, independently of the formula's own code:

* completed lattice: when the ghosts are exactly the lattice sites missing from a particle's
  support and the target density is the complete lattice's, the estimate is 1;
* ghost doubling: two ghosts at every ghost position halve the estimate;
* flat wall with the ghost row on the first missing lattice row: the estimate is the ratio of the
  ghost spacing to the fluid spacing, dg / s (the two kernel sums are Riemann sums of the same
  line integral at spacings s and dg) -- 0.512 for the paper's tank, Table 2's gamma1 = 0.5;
* density_parts agrees with density (independently pinned) for any gamma1.
"""
import math

import numpy as np

import oracle as O
import sph_inputs as si


def _lattice(s, nx, ny, y0=0.0):
    xs = np.arange(-nx, nx + 1) * s
    ys = y0 - np.arange(0, ny) * s
    X, Y = np.meshgrid(xs, ys)
    return np.stack([X.ravel(), Y.ravel()], 1)


def test_completed_lattice_gives_one():
    sp = si.preset(1.0)
    s = sp.spacing
    full = np.stack(np.meshgrid(np.arange(-12, 13) * s, np.arange(-12, 13) * s), -1).reshape(-1, 2)
    fluid = full[full[:, 1] <= 0.0]
    ghost = full[full[:, 1] > 0.0]
    rho_full, _ = O.density(sp.__class__(**{**sp.as_dict(), "gamma1": 0.0}), full, np.zeros((0, 2)))
    i0 = np.argmin(np.abs(full).sum(1))                     # the centre site: full support
    _, g, sf, sg = O.estimate_gamma1(sp, fluid, ghost, rho_target=rho_full[i0])
    near = (np.abs(fluid[:, 0]) <= 4 * s) & (fluid[:, 1] >= -s) & (sg > 0)
    assert near.sum() >= 9
    assert np.allclose(g[near], 1.0, rtol=0, atol=1e-12)


def test_ghost_doubling_halves():
    t = si.make_tank(1.0)
    gp, _ = O.ghosts(t.ghost_b, np.zeros(6))
    w1, g1, _, _ = O.estimate_gamma1(t.params, t.pos, gp)
    w2, g2, _, _ = O.estimate_gamma1(t.params, t.pos, np.concatenate([gp, gp]))
    ok = np.isfinite(g1)
    assert ok.sum() > 20 and np.array_equal(ok, np.isfinite(g2))
    assert np.allclose(g2[ok], 0.5 * g1[ok], rtol=1e-12, atol=0)
    assert abs(w2 - 0.5 * w1) <= 1e-12 * abs(w1)


def test_flat_wall_template_is_spacing_ratio():
    """The paper's wall: ghosts 2 pi R / 236 = 5.32 mm apart, fluid lattice s = 10.39 mm (reading
    R1), the ghost row where the first missing fluid row would be (distance s from the first
    fluid row).  Only that row lies within 2h of the fluid (2h = 1.81 s), so the estimate is
    sum_k W(k s) / sum_k W(k dg) -> dg / s; measured within the Riemann-sum error (< 1 %)."""
    sp = si.preset(1.0)
    s = sp.spacing
    dg = 2.0 * math.pi * sp.R / si.N_GHOST_PAPER
    fluid = _lattice(s, 40, 12, y0=-s)
    kg = int(40 * s / dg)
    ghost = np.stack([np.arange(-kg, kg + 1) * dg, np.zeros(2 * kg + 1)], 1)
    _, g, sf, sg = O.estimate_gamma1(sp, fluid, ghost)
    centre = (np.abs(fluid[:, 0]) <= 5 * s) & np.isfinite(g)
    assert centre.sum() >= 11
    assert np.all(np.abs(fluid[centre, 1] + s) < 1e-12)   # only the first row sees the wall
    assert np.allclose(g[centre], dg / s, rtol=1e-2)
    assert abs(dg / s - 0.5) < 0.02                        # Table 2: gamma1 = 0.5


def test_density_parts_match_density():
    t = si.moving_tank(1.0, seed=9, vel=0.0)
    gp, _ = O.ghosts(t.ghost_b, np.zeros(6))
    sf, sg = O.density_parts(t.params, t.pos, gp)
    for g1 in (0.0, 0.5, 1.7):
        sp = t.params.__class__(**{**t.params.as_dict(), "gamma1": g1})
        rho, _ = O.density(sp, t.pos, gp)
        assert np.allclose(rho, sp.mass * (sf + g1 * sg), rtol=1e-13, atol=0)
    # at the estimate, each wall particle's density is the target
    _, g, _, _ = O.estimate_gamma1(t.params, t.pos, gp)
    i = np.flatnonzero(np.isfinite(g))[:5]
    for k in i:
        sp = t.params.__class__(**{**t.params.as_dict(), "gamma1": g[k]})
        rho, _ = O.density(sp, t.pos, gp)
        assert abs(rho[k] - sp.rho0) <= 1e-11 * sp.rho0


def test_tank_wall_layer_estimate():
    """On the C1 rest lattice the wall-layer estimate is close to Table 2's 0.5 (0.517)."""
    t = si.make_tank(1.0)
    gp, _ = O.ghosts(t.ghost_b, np.zeros(6))
    wall, g, _, sg = O.estimate_gamma1(t.params, t.pos, gp)
    assert 0.45 <= wall <= 0.6
    assert np.isfinite(g).sum() == (sg > 0).sum() > 50
