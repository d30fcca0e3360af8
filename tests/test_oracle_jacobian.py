"""Pins of the oracle's linearization (P:259 item 2; SPEC
linearization module): the central-difference Jacobian of the continuous-time f is checked
against closed forms and exact identities of the mathematics, not against itself.

* rigid-only tank: f is linear, A and B are known in closed form (Eq. tankdynamics);
* kinematic block d(pos)/dt = vel: exact identity / zero pattern;
* linear momentum: sum_i m a_i + m_B rdd = u for every x (internal forces cancel in pairs,
  fluid-ghost reactions go to the body), so the momentum-weighted column sums of A vanish and
  those of B are the identity;
* angular momentum: sum_i m x_i x a_i + m_B r x rdd + J thdd = r x u + tau for every x (central
  pair forces, reactions with their arms); its derivative gives one exact identity per column;
* translation, Galilean (uniform velocity) and rotation invariance of f;
* spectra of real matrices are closed under conjugation.
"""
import math

import numpy as np
import pytest

import oracle as O
import sph_inputs as si

BODY = [0.05, -0.03, 0.4, 0.01, -0.02, 0.05]


@pytest.fixture(scope="module")
def lin_c1():
    t = si.moving_tank(1.0, seed=3, vel=0.02, body=BODY)
    x = O.state_vector(t.pos, t.vel, t.body)
    u = (5.0, 2.0, 1.0)
    A, B = O.jacobian_fd(t.params, x, t.ghost_b, u)
    f = O.deriv(t.params, x, t.ghost_b, u)
    return t, x, u, A, B, f


def _blocks(n):
    return dict(pos=slice(0, 2 * n), vel=slice(2 * n, 4 * n), r=slice(4 * n, 4 * n + 2),
                th=4 * n + 2, rd=slice(4 * n + 3, 4 * n + 5), thd=4 * n + 5)


def test_rigid_only_jacobian_closed_form():
    t = si.make_tank(1.0)
    sp = t.params
    x = O.state_vector(np.zeros((0, 2)), np.zeros((0, 2)), np.array([0.1, -0.2, 0.3, 0.01, 0.02, 0.03]))
    A, B = O.jacobian_fd(sp, x, t.ghost_b, (5.0, 2.0, 1.0))
    A_ref = np.zeros((6, 6))
    A_ref[0, 3] = A_ref[1, 4] = A_ref[2, 5] = 1.0
    B_ref = np.zeros((6, 3))
    B_ref[3, 0] = B_ref[4, 1] = 1.0 / sp.m_body
    B_ref[5, 2] = 1.0 / sp.J_body
    assert np.allclose(A, A_ref, rtol=0, atol=1e-9)          # FD rounding eps / h_rel
    assert np.allclose(B, B_ref, rtol=1e-9, atol=1e-15)
    ev = np.linalg.eigvals(A)
    assert np.abs(ev).max() < 1e-9                               # nilpotent (double integrators)


def test_kinematic_block_exact(lin_c1):
    t, x, u, A, B, f = lin_c1
    n = t.n_fluid
    b = _blocks(n)
    # unit entries up to the difference quotient's rounding (eps / h_rel), zeros exact
    assert np.allclose(A[b["pos"], b["vel"]], np.eye(2 * n), rtol=0, atol=1e-9)
    assert not (A[b["pos"], b["vel"]] * (1 - np.eye(2 * n))).any()
    assert not A[b["pos"], :2 * n].any() and not A[b["pos"], 4 * n:].any()
    assert not B[b["pos"]].any()
    for row, col in ((4 * n, 4 * n + 3), (4 * n + 1, 4 * n + 4), (4 * n + 2, 4 * n + 5)):
        e = np.zeros(4 * n + 6)
        e[col] = 1.0
        assert np.allclose(A[row], e, rtol=0, atol=1e-9) and np.count_nonzero(A[row]) == 1


def test_state_is_active(lin_c1):
    """The linearization point exercises every term: wall contacts in both viscous branches,
    a moving and spinning body."""
    t, x, u, A, B, f = lin_c1
    n = t.n_fluid
    gp, gv = O.ghosts(t.ghost_b, t.body)
    h = t.params.h
    d2 = ((t.pos[:, None, :] - gp[None, :, :]) ** 2).sum(-1)
    i, g = np.nonzero(d2 < h * h)
    vr = ((t.vel[i] - gv[g]) * (t.pos[i] - gp[g])).sum(-1)
    assert (vr < 0).sum() > 5 and (vr > 0).sum() > 5
    assert np.abs(A[4 * n + 3:, 4 * n:4 * n + 6]).max() > 0     # body couples to its own pose


def test_linear_momentum_identity(lin_c1):
    t, x, u, A, B, f = lin_c1
    sp = t.params
    n = t.n_fluid
    m = sp.mass
    for c in range(2):
        rows = np.arange(2 * n + c, 4 * n, 2)
        colsum_A = m * A[rows].sum(0) + sp.m_body * A[4 * n + 3 + c]
        colsum_B = m * B[rows].sum(0) + sp.m_body * B[4 * n + 3 + c]
        scale = m * np.abs(A[rows]).max()
        assert np.abs(colsum_A).max() <= 1e-6 * scale, np.abs(colsum_A).max() / scale
        e = np.zeros(3)
        e[c] = 1.0
        assert np.allclose(colsum_B, e, atol=1e-8)
    # and the identity itself at the point: sum m a + m_B rdd = u
    acc = f[2 * n:4 * n].reshape(-1, 2)
    tot = m * acc.sum(0) + sp.m_body * f[4 * n + 3:4 * n + 5]
    assert np.allclose(tot, u[:2], atol=1e-9 * m * np.abs(acc).sum())


def test_angular_momentum_identity(lin_c1):
    """d/dx_j of  sum_i m x_i x a_i + m_B r x rdd + J thdd - r x u  = 0  for every column j."""
    t, x, u, A, B, f = lin_c1
    sp = t.params
    n = t.n_fluid
    m, mb, J = sp.mass, sp.m_body, sp.J_body
    pos = x[:2 * n].reshape(-1, 2)
    acc = f[2 * n:4 * n].reshape(-1, 2)
    r = x[4 * n:4 * n + 2]
    rdd = f[4 * n + 3:4 * n + 5]
    cross = lambda a, b: a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]
    L0 = m * cross(pos, acc).sum() + mb * cross(r, rdd) + J * f[4 * n + 5] - cross(r, np.array(u[:2]))
    assert abs(L0 - u[2]) <= 1e-9 * m * np.abs(pos).max() * np.abs(acc).sum()
    dA = A[2 * n:4 * n].reshape(n, 2, -1)                       # d a_i / dx_j
    ident = np.zeros(4 * n + 6)
    # explicit dependence on positions (d x_i/dx_j = e) and on r
    for c, sgn in ((0, 1.0), (1, -1.0)):                       # e_x x a = a_y, e_y x a = -a_x
        ident[c:2 * n:2] += m * sgn * acc[:, 1 - c]
        ident[4 * n + c] += mb * sgn * rdd[1 - c] - sgn * u[1 - c]
    ident += m * (pos[:, 0, None] * dA[:, 1] - pos[:, 1, None] * dA[:, 0]).sum(0)
    ident += mb * (r[0] * A[4 * n + 4] - r[1] * A[4 * n + 3]) + J * A[4 * n + 5]
    scale = m * np.abs(pos).max() * np.abs(dA).max()
    assert np.abs(ident).max() <= 1e-6 * scale, np.abs(ident).max() / scale


def _matvec_err(M, v, want):
    """max |M v - want| relative to the natural scale max_i sum_j |M_ij v_j| of the product
    (the identities cancel large terms; the FD error of each entry scales with it)."""
    return np.abs(M @ v - want).max() / (np.abs(M) @ np.abs(v)).max()


def test_translation_galilean_rotation_invariance(lin_c1):
    t, x, u, A, B, f = lin_c1
    n = t.n_fluid
    acc_rows = np.r_[2 * n:4 * n, 4 * n + 3:4 * n + 6]
    for c in range(2):
        tr = np.zeros(4 * n + 6)                                  # translate everything
        tr[c:2 * n:2] = 1.0
        tr[4 * n + c] = 1.0
        assert _matvec_err(A[acc_rows], tr, 0.0) <= 1e-6
        gal = np.zeros(4 * n + 6)                                 # uniform velocity shift
        gal[2 * n + c:4 * n:2] = 1.0
        gal[4 * n + 3 + c] = 1.0
        assert _matvec_err(A[acc_rows], gal, 0.0) <= 1e-6
    # rotation about the origin (u = 0): f(R x) = R f(x) => A (Jx) = J f
    tz = si.moving_tank(1.0, seed=3, vel=0.02, body=BODY)
    x0 = O.state_vector(tz.pos, tz.vel, tz.body)
    A0, _ = O.jacobian_fd(tz.params, x0, tz.ghost_b, (0.0, 0.0, 0.0))
    f0 = O.deriv(tz.params, x0, tz.ghost_b, (0.0, 0.0, 0.0))
    rot = lambda v: np.stack([-v[..., 1], v[..., 0]], -1)        # z x v
    gen = np.concatenate([rot(x0[:2 * n].reshape(-1, 2)).ravel(), rot(x0[2 * n:4 * n].reshape(-1, 2)).ravel(),
                          rot(x0[4 * n:4 * n + 2]), [1.0], rot(x0[4 * n + 3:4 * n + 5]), [0.0]])
    want = np.concatenate([rot(f0[:2 * n].reshape(-1, 2)).ravel(), rot(f0[2 * n:4 * n].reshape(-1, 2)).ravel(),
                           rot(f0[4 * n:4 * n + 2]), [0.0], rot(f0[4 * n + 3:4 * n + 5]), [0.0]])
    assert _matvec_err(A0, gen, want) <= 1e-6


def test_fd_step_convergence(lin_c1):
    """Central differences at the default step h = 1e-7 and at 2h agree to 1e-8 of max|A| (no
    stencil straddles a kink of f, no rounding plateau)."""
    t, x, u, A, B, f = lin_c1
    A2, _ = O.jacobian_fd(t.params, x, t.ghost_b, u, h_rel=2e-7)
    assert np.abs(A2 - A).max() <= 1e-8 * np.abs(A).max()


def test_spectrum_conjugate_symmetric(lin_c1):
    t, x, u, A, B, f = lin_c1
    ev = np.linalg.eigvals(A)
    a = np.sort_complex(ev)
    b = np.sort_complex(np.conj(ev))
    assert np.allclose(a, b, atol=1e-8 * np.abs(ev).max())
    assert np.abs(ev.imag).max() > 0                              # oscillatory modes present
