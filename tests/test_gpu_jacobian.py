"""GPU linearization (sph_jacobian) vs the oracle's central-difference
Jacobian (tests/test_oracle_jacobian.py pins it), plus the exact identities the analytic
(forward-mode) Jacobian must satisfy to rounding."""
import numpy as np
import pytest

import oracle as O
import sph_inputs as si

pytestmark = pytest.mark.gpu

BODY = [0.05, -0.03, 0.4, 0.01, -0.02, 0.05]


def _ctx(t, B=1, **kw):
    from paper_2604_12505_b200 import SphContext
    return SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=B, **kw)


def _point(ctx, b=0):
    pv = ctx.get_particles(b).astype(np.float64)
    body = ctx.get_body_state()[b]
    return O.state_vector(pv[:, :2], pv[:, 2:], body)


def _block_err(Ag, Ao, n):
    """max over the natural blocks of max|Ag - Ao| / max|Ao| (per block)."""
    rows = {"pos": slice(0, 2 * n), "acc": slice(2 * n, 4 * n), "body": slice(4 * n, 4 * n + 6)}
    cols = {"pos": slice(0, 2 * n), "vel": slice(2 * n, 4 * n), "body": slice(4 * n, 4 * n + 6)}
    worst = 0.0
    for rs in rows.values():
        for cs in cols.values():
            ref = np.abs(Ao[rs, cs]).max()
            if ref > 0:
                worst = max(worst, np.abs(Ag[rs, cs] - Ao[rs, cs]).max() / ref)
            else:
                assert np.abs(Ag[rs, cs]).max() == 0.0
    return worst


@pytest.mark.parametrize("case", ["moving_rotated", "after_actuated_steps", "clamped_eos"])
def test_jacobian_matches_oracle_fd(case):
    over = dict(clamp_negative_pressure=1.0) if case == "clamped_eos" else {}
    t = si.moving_tank(1.0, seed=3, vel=0.02, body=BODY, **over)
    ctx = _ctx(t)
    ctx.set_body_state(np.array([BODY]))
    if case == "after_actuated_steps":
        ctx.step(np.array([[5.0, 2.0, 1.0]], np.float32), 30)
    x = _point(ctx)
    A, B = ctx.jacobian(0)
    Ao, Bo = O.jacobian_fd(t.params, x, t.ghost_b, (5.0, 2.0, 1.0))
    n = t.n_fluid
    assert A.shape == (4 * n + 6, 4 * n + 6) and B.shape == (4 * n + 6, 3)
    # the oracle's central differences are accurate to ~2e-9 of max|A| (its step-convergence
    # pin); the analytic float64 Jacobian agrees to that level
    assert _block_err(A, Ao, n) <= 5e-7       # per block: FD rounding floor of small blocks
    # B is exact on the GPU (test_jacobian_exact_identities); the oracle's central differences
    # carry a rounding floor ~eps |f| / h_step, larger where the wall force is larger
    assert np.abs(B - Bo).max() <= 1e-7 * np.abs(Bo).max()
    ctx.close()


def test_jacobian_exact_identities():
    """Momentum balance and invariances hold for the analytic Jacobian to rounding."""
    t = si.moving_tank(1.0, seed=5, vel=0.02, body=BODY)
    ctx = _ctx(t)
    ctx.set_body_state(np.array([BODY]))
    A, B = ctx.jacobian(0)
    sp = t.params
    n = t.n_fluid
    m = sp.mass
    for c in range(2):
        rows = np.arange(2 * n + c, 4 * n, 2)
        colsum = m * A[rows].sum(0) + sp.m_body * A[4 * n + 3 + c]
        assert np.abs(colsum).max() <= 1e-11 * m * np.abs(A[rows]).max()
        tr = np.zeros(4 * n + 6)
        tr[c:2 * n:2] = 1.0
        tr[4 * n + c] = 1.0
        acc_rows = np.r_[2 * n:4 * n, 4 * n + 3:4 * n + 6]
        assert np.abs(A[acc_rows] @ tr).max() <= 1e-11 * (np.abs(A[acc_rows]) @ np.abs(tr)).max()
        gal = np.zeros(4 * n + 6)
        gal[2 * n + c:4 * n:2] = 1.0
        gal[4 * n + 3 + c] = 1.0
        assert np.abs(A[acc_rows] @ gal).max() <= 1e-11 * (np.abs(A[acc_rows]) @ np.abs(gal)).max()
    assert np.array_equal(A[:2 * n, 2 * n:4 * n], np.eye(2 * n))   # kinematic block, exact
    Bref = np.zeros((4 * n + 6, 3))
    Bref[4 * n + 3, 0] = Bref[4 * n + 4, 1] = 1.0 / sp.m_body
    Bref[4 * n + 5, 2] = 1.0 / sp.J_body
    assert np.array_equal(B, Bref)
    ctx.close()


def test_rigid_only_and_device_pointers():
    import torch
    t = si.make_tank(1.0)
    t0 = si.Tank(t.params, np.zeros((0, 2)), np.zeros((0, 2)), t.ghost_b)
    ctx = _ctx(t0)
    A, B = ctx.jacobian(0)
    Aref = np.zeros((6, 6))
    Aref[0, 3] = Aref[1, 4] = Aref[2, 5] = 1.0
    assert np.array_equal(A, Aref)
    assert B[3, 0] == 1.0 / t.params.m_body and B[5, 2] == 1.0 / t.params.J_body
    ctx.close()
    tm = si.moving_tank(1.0, seed=3, vel=0.02, body=BODY)
    ctx = _ctx(tm, B=2)
    ctx.set_body_state(np.array([BODY, BODY]))
    Ah, Bh = ctx.jacobian(1)
    Ad, Bd = ctx.jacobian(1, device=True)
    assert isinstance(Ad, torch.Tensor) and Ad.is_cuda
    assert np.array_equal(Ah, Ad.cpu().numpy()) and np.array_equal(Bh, Bd.cpu().numpy())
    ctx.close()


def test_eigen_trace_spectra():
    """Figs. 5-6 analysis: spectra along an actuated C1 trajectory are conjugate-
    symmetric, agree with the spectrum of the oracle's Jacobian at the same point, and vary in
    time (the nonlinearity the paper points out)."""
    from paper_2604_12505_b200.linearize import eigen_trace
    t = si.make_tank(1.0)
    s = O.settle(t, seconds=2.0)
    ts = si.Tank(t.params, s.pos, s.vel, t.ghost_b).snapped()
    ctx = _ctx(ts)
    u = np.zeros((1, 4, 3), np.float32)
    u[0, :, 0] = 40.0                                              # strong push: sloshing starts
    u[0, :, 2] = 5.0
    times, spectra = eigen_trace(ctx, u, stride=2)
    assert len(spectra) == 2 and times[1] > times[0]
    for ev in spectra:
        a = np.sort_complex(ev)
        assert np.allclose(a, np.sort_complex(np.conj(ev)), atol=1e-7 * np.abs(ev).max())
    dist = np.abs(np.sort_complex(spectra[0]) - np.sort_complex(spectra[1])).max()
    assert dist > 0
    # last point: compare with numpy's eigenvalues of the oracle FD Jacobian
    x = _point(ctx)
    Ao, _ = O.jacobian_fd(ts.params, x, ts.ghost_b)
    A, _ = ctx.jacobian(0)
    ev_g = np.sort_complex(np.linalg.eigvals(A))
    ev_o = np.sort_complex(np.linalg.eigvals(Ao))
    assert np.abs(ev_g.real.max() - ev_o.real.max()) <= 1e-4 * np.abs(ev_o).max()
    assert np.abs(np.abs(ev_g).max() - np.abs(ev_o).max()) <= 1e-6 * np.abs(ev_o).max()
    ctx.close()


def test_eigenvalues_library_solver():
    """sph_eigenvalues (cuSOLVER Xgeev): SPEC linearization examples (zero matrix -> 0,
    companion of xdd = -x -> +-i) and a random matrix against LAPACK (numpy)."""
    import torch
    t = si.make_tank(1.0)
    ctx = _ctx(t)
    assert np.allclose(ctx.eigenvalues(np.zeros((4, 4))), 0.0)
    ev = np.sort_complex(ctx.eigenvalues(np.array([[0.0, 1.0], [-1.0, 0.0]])))
    assert np.allclose(ev, [-1j, 1j], atol=1e-14)
    rng = np.random.Generator(np.random.Philox(7))
    M = rng.normal(size=(300, 300))
    ev = ctx.eigenvalues(M)
    ref = np.linalg.eigvals(M)
    # match each LAPACK eigenvalue to its nearest GPU eigenvalue
    d = np.abs(ref[:, None] - ev[None, :]).min(1)
    assert d.max() <= 1e-10 * np.abs(ref).max()
    evd = ctx.eigenvalues(torch.from_numpy(M).cuda())
    assert evd.is_cuda and np.allclose(np.sort_complex(evd.cpu().numpy()), np.sort_complex(ev), atol=1e-12)
    ctx.close()


def test_jacobian_scratch_growth_keeps_gamma1_buffer_valid():
    """Scratch ownership on one context: gamma1 estimate -> Jacobian (device pointers) ->
    Jacobian (host pointers: larger scratch, re-allocated) -> gamma1 estimate.  The gamma1
    reduction buffer must survive the Jacobian's scratch growth (no use after free): both
    estimates are identical, and so are both Jacobians."""
    t = si.moving_tank(1.0, seed=5, vel=0.01)
    ctx = _ctx(t)
    w0, g0, s0 = ctx.gamma1_estimate(0)
    Ad, Bd = ctx.jacobian(0, device=True)
    Ah, Bh = ctx.jacobian(0, device=False)
    w1, g1, s1 = ctx.gamma1_estimate(0)
    assert np.isfinite(w0) and w0 == w1
    assert np.array_equal(s0, s1) and np.array_equal(np.isnan(g0), np.isnan(g1))
    assert np.array_equal(Ad.cpu().numpy(), Ah) and np.array_equal(Bd.cpu().numpy(), Bh)
    ctx.close()
