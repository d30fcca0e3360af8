"""Pins of the oracle's neighbour sets, density, pressure and forces.  P:n = PAPER.md line n."""
import json
import os

import numpy as np
import pytest

import oracle as O
import sph_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _sets(off, idx):
    return [tuple(idx[off[i]:off[i + 1]]) for i in range(len(off) - 1)]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_cell_list_equals_brute_force(seed):
    """Footnote P:135: neighbours within the support.  Cell-list sets == O(N^2) brute force."""
    t = si.random_tank(700, 60, seed=seed, R=0.06)
    a = O.neighbours(t.params, t.pos, use_cells=False)
    b = O.neighbours(t.params, t.pos, use_cells=True)
    assert _sets(*a) == _sets(*b)
    # lattice (many near-ties at the support radius)
    t = si.make_tank(1.0, jitter=0.01, seed=seed)
    a = O.neighbours(t.params, t.pos, use_cells=False)
    b = O.neighbours(t.params, t.pos, use_cells=True)
    assert _sets(*a) == _sets(*b)


def test_float32_predicates_match_numpy_float32():
    """Reading A19: float32 predicate dx*dx + dy*dy < H*H and cell = floor((x - o) * inv) with
    IEEE single ops; reproduced with numpy float32 arithmetic (no contraction in numpy)."""
    t = si.random_tank(400, 80, seed=5, R=0.05)
    p32 = t.pos.astype(np.float32)
    H = np.float32(2 * t.params.h)
    H2 = np.float32(H * H)
    off, idx = O.neighbours_f32(p32, H2)
    dx = p32[:, None, 0] - p32[None, :, 0]
    dy = p32[:, None, 1] - p32[None, :, 1]
    d2 = (dx * dx) + (dy * dy)
    assert d2.dtype == np.float32
    m = d2 < H2
    np.fill_diagonal(m, False)
    ref = [tuple(np.nonzero(m[i])[0]) for i in range(len(p32))]
    assert _sets(off, idx) == ref
    g32 = (si.ghost_ring(80, 0.05) * 1.0).astype(np.float32)
    h2 = np.float32(np.float32(t.params.h) * np.float32(t.params.h))
    off, idx = O.ghost_neighbours_f32(p32, g32, h2)
    dx = p32[:, None, 0] - g32[None, :, 0]
    dy = p32[:, None, 1] - g32[None, :, 1]
    m = ((dx * dx) + (dy * dy)) < h2
    assert _sets(off, idx) == [tuple(np.nonzero(m[i])[0]) for i in range(len(p32))]
    inv = np.float32(1.0) / H
    ox, oy = np.float32(-0.07), np.float32(-0.0712)
    cells = O.cells_f32(p32, ox, oy, inv)
    ref = np.floor(((p32 - np.array([ox, oy], np.float32)) * inv)).astype(np.int32)
    assert np.array_equal(cells, ref)


def test_golden_two_fluid_particles():
    """density, EOS pressure and accelerations of a 2-particle system (no ghosts)."""
    g = json.load(open(os.path.join(GOLD, "g1_two_fluid.json")))
    sp = si.preset(1.0)
    pos, vel = np.array(g["pos"]), np.array(g["vel"])
    rho, P = O.density(sp, pos, np.zeros((0, 2)))
    tol = g["rel_tol"]
    assert rho == pytest.approx([g["rho"]] * 2, rel=tol)
    assert P == pytest.approx([g["P"]] * 2, rel=tol)
    acc, Fb, Tb = O.forces(sp, pos, vel, rho, P, np.zeros((0, 2)), np.zeros((0, 2)), np.zeros(6))
    assert acc[0] == pytest.approx(g["a1"], rel=tol)
    assert acc[1] == pytest.approx([-g["a1"][0], -g["a1"][1]], rel=tol)
    assert Fb.tolist() == [0.0, 0.0] and Tb == 0.0


def test_golden_fluid_ghost():
    """ghost kinematics, wall density term, wall force and body torque."""
    g = json.load(open(os.path.join(GOLD, "g2_fluid_ghost.json")))
    sp = si.preset(1.0)
    body = np.array(g["body"])
    gp, gv = O.ghosts(np.array(g["ghost_b"]), body)
    tol = g["rel_tol"]
    assert gp[0] == pytest.approx(g["ghost_pos"], rel=tol)
    assert gv[0] == pytest.approx(g["ghost_vel"], rel=tol)
    pos, vel = np.array(g["pos"]), np.array(g["vel"])
    rho, P = O.density(sp, pos, gp)
    assert rho[0] == pytest.approx(g["rho"], rel=tol)
    assert P[0] == pytest.approx(g["P"], rel=tol)
    acc, Fb, Tb = O.forces(sp, pos, vel, rho, P, gp, gv, body)
    assert acc[0] * sp.mass == pytest.approx(g["G"], rel=tol)
    assert Fb == pytest.approx([-g["G"][0], -g["G"][1]], rel=tol)
    assert Tb == pytest.approx(g["T_body"], rel=tol)


def test_isolated_particle_density_and_eos():
    """Only the self term: rho = m W_cb(0); EOS P = k (rho - rho0):
    rho = rho0 => P = 0; k = 3, rho = rho0 + 1 => P = 3."""
    sp = si.preset(1.0)
    rho, P = O.density(sp, np.array([[0.0, 0.0]]), np.zeros((0, 2)))
    assert rho[0] == sp.mass * O.W_cb(sp, 0.0)
    assert P[0] == pytest.approx(3.0 * (rho[0] - 1017.0), rel=1e-15)
    # choose mass so the self density is exactly rho0 (+1): P = 0 (3)
    for target, want in ((1017.0, 0.0), (1018.0, 3.0)):
        sp2 = si.preset(1.0, mass=target / O.W_cb(sp, 0.0))
        _, P = O.density(sp2, np.array([[0.0, 0.0]]), np.zeros((0, 2)))
        assert P[0] == pytest.approx(want, abs=1e-9)


def test_square_lattice_interior_density():
    """Kernel normalisation => interior density of a uniform lattice ~ rho0.  Reading R1
    (spacing s = sqrt(3) 6 mm, m = rho0 s^2): the finite square-lattice sum gives
    rho/rho0 = s^2 sum W = 0.99967967 (SURVEY 8(c) pin table)."""
    sp = si.preset(1.0)
    s = sp.spacing
    n = 9
    ii = np.arange(-n, n + 1) * s
    X, Y = np.meshgrid(ii, ii)
    pos = np.stack([X.ravel(), Y.ravel()], 1)
    rho, _ = O.density(sp, pos, np.zeros((0, 2)))
    centre = np.argmin(np.hypot(pos[:, 0], pos[:, 1]))
    assert rho[centre] / sp.rho0 == pytest.approx(0.99967967, abs=5e-9)
    assert abs(rho[centre] / sp.rho0 - 1.0) < 3.3e-4


def test_pair_forces_are_newton_pairs():
    """Eq. momentum is symmetric (momentum exactly conserved); sum of internal forces = 0."""
    t = si.random_tank(300, 0, seed=11, R=0.04, vel_scale=0.05)
    sp = t.params
    rho, P = O.density(sp, t.pos, np.zeros((0, 2)))
    acc, _, _ = O.forces(sp, t.pos, t.vel, rho, P, np.zeros((0, 2)), np.zeros((0, 2)), np.zeros(6))
    tot = (sp.mass * acc).sum(0)
    scale = (sp.mass * np.abs(acc)).sum()
    assert np.all(np.abs(tot) < 1e-13 * scale)
    # angular: sum r_i x F_i = 0 for central pair forces
    L = (t.pos[:, 0] * acc[:, 1] - t.pos[:, 1] * acc[:, 0]).sum() * sp.mass
    assert abs(L) < 1e-13 * scale * 0.04


def test_viscosity_vanishes_for_uniform_velocity():
    """Eq. viscous depends on rdot_ij only."""
    t = si.random_tank(200, 0, seed=3, R=0.03)
    sp = t.params
    rho, P = O.density(sp, t.pos, np.zeros((0, 2)))
    z = np.zeros((0, 2))
    a0, _, _ = O.forces(sp, t.pos, np.zeros_like(t.pos), rho, P, z, z, np.zeros(6))
    a1, _, _ = O.forces(sp, t.pos, np.tile([0.3, -0.2], (200, 1)), rho, P, z, z, np.zeros(6))
    assert np.allclose(a0, a1, rtol=0, atol=1e-12 * np.abs(a0).max())


def test_compressed_pair_repels_and_closing_pair_is_damped():
    """Physics signs fixed by the paper: P > 0 (rho > rho0) pushes particles apart (-F^p in
    Alg. 1 l.8); artificial viscosity opposes approach (Monaghan 1983)."""
    sp = si.preset(1.0, mass=1017.0 / 4000.0)   # tiny mass -> make rho > rho0 by crowding
    # a crowded cluster: everybody compressed
    g = np.arange(-3, 4) * 0.3 * sp.h
    X, Y = np.meshgrid(g, g)
    pos = np.stack([X.ravel(), Y.ravel()], 1)
    rho, P = O.density(sp, pos, np.zeros((0, 2)))
    assert np.all(P > 0)
    z = np.zeros((0, 2))
    acc, _, _ = O.forces(sp, pos, np.zeros_like(pos), rho, P, z, z, np.zeros(6))
    outward = (acc * pos).sum(1)
    edge = np.hypot(pos[:, 0], pos[:, 1]) > 0.5 * g.max()
    assert np.all(outward[edge] > 0)
    # closing pair (pressure switched off via k = 0): viscous acceleration opposes approach
    sp0 = si.preset(1.0, k=0.0)
    pos = np.array([[0.0, 0.0], [0.6 * sp.h, 0.0]])
    vel = np.array([[0.1, 0.0], [-0.1, 0.0]])
    rho, P = O.density(sp0, pos, z)
    acc, _, _ = O.forces(sp0, pos, vel, rho, P, z, z, np.zeros(6))
    assert acc[0, 0] < 0 < acc[1, 0]


def test_wall_pressure_repels_and_wall_viscosity_is_one_sided():
    """Reading A4: a compressed particle near a ghost is pushed away from the wall.
    Eq. viscous_b2f uses min(v.r, 0): a separating particle feels no wall viscosity."""
    sp = si.preset(1.0, k=3.0, alpha=0.0)
    gpos = np.array([[0.2, 0.0]])
    pos = np.array([[0.2 - 0.4 * sp.h, 0.0]])
    z = np.zeros((1, 2))
    rho = np.array([1100.0])
    P = sp.k * (rho - sp.rho0)
    acc, Fb, _ = O.forces(sp, pos, z, rho, P, gpos, z, np.zeros(6))
    assert acc[0, 0] < 0 and Fb[0] > 0       # fluid pushed inward, wall pushed outward
    sp_b = si.preset(1.0, k=0.0)
    P0 = np.zeros(1)
    a_sep, _, _ = O.forces(sp_b, pos, np.array([[-0.05, 0.0]]), rho, P0, gpos, z, np.zeros(6))
    assert np.all(a_sep == 0.0)
    a_app, _, _ = O.forces(sp_b, pos, np.array([[0.05, 0.0]]), rho, P0, gpos, z, np.zeros(6))
    assert a_app[0, 0] < 0
