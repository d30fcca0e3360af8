"""Pins of the LPV surrogate oracle (oracle/lpv.py) against what is fixed
independently of its code: library LTI simulation (scipy.signal.dlsim) where the model collapses
to an LTI system, closed forms of the BFR footnote, the regularization's exact gradient,
step convergence of the central differences, and the cumulative-sum form of Eq. (28)."""
import numpy as np
import scipy.signal as sig

from oracle import lpv as L


def _rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def _theta(seed, scale=0.3):
    r = _rng(seed)
    P = {n: r.normal(0, scale, s) for n, s in L.SIZES}
    P["A0"] = 0.9 * np.eye(4) + r.normal(0, 0.03, (4, 4))
    P["A1"] = r.normal(0, 0.02, (4, 4))
    return P


def _dlsim(A, B, C, u, x0):
    _, y, _ = sig.dlsim((A, B, C, np.zeros((3, 3)), 0.05), u, x0=x0)
    return y


def test_count_and_pack_roundtrip():
    assert L.N_THETA == 137
    P = _theta(1)
    th = L.pack(P)
    Q = L.unpack(th)
    for n, _ in L.SIZES:
        assert np.array_equal(Q[n], P[n])


def test_lti_collapse_matches_dlsim():
    P = _theta(2)
    for n in ("A1", "B1", "C1"):
        P[n] = np.zeros_like(P[n])
    u = _rng(3).normal(size=(60, 3))
    x0 = _rng(4).normal(size=4)
    yh, _ = L.simulate(L.pack(P), x0, u)
    assert np.allclose(yh, _dlsim(P["A0"], P["B0"], P["C0"], u, x0), rtol=1e-12, atol=1e-13)


def test_saturated_scheduling_is_frozen_lti():
    """b1 = +-50 saturates layer 1 at sign(b1) whatever the input; W2 h1 + b2 then has a sign
    fixed by hand, so p is a known constant and the model is the frozen LTI M0 + p M1."""
    P = _theta(5)
    P["W1"] = 1e-3 * P["W1"]
    P["b1"] = np.array([50.0, -50.0, 50.0, 50.0])
    P["W2"] = np.array([[30.0, 0, 0, 0], [0, 30.0, 0, 0], [0, 0, -30.0, 0], [10.0, 10.0, 10.0, 10.0]])
    P["b2"] = np.zeros(4)
    # h1 = (1, -1, 1, 1) -> W2 h1 = (30, -30, -30, 20) -> h2 = (1, -1, -1, 1)
    P["W3"] = np.array([[0.2, 0.1, -0.3, 0.05]])
    P["b3"] = np.array([0.4])
    p = 0.2 - 0.1 + 0.3 + 0.05 + 0.4
    u = _rng(6).normal(size=(50, 3))
    x0 = _rng(7).normal(size=4)
    yh, _ = L.simulate(L.pack(P), x0, u)
    ref = _dlsim(P["A0"] + p * P["A1"], P["B0"] + p * P["B1"], P["C0"] + p * P["C1"], u, x0)
    assert np.allclose(yh, ref, rtol=1e-12, atol=1e-12)


def test_zero_input_zero_state():
    yh, x = L.simulate(L.pack(_theta(8)), np.zeros(4), np.zeros((20, 3)))
    assert np.all(yh == 0.0) and np.all(x == 0.0)


def test_bfr_closed_forms():
    y = _rng(9).normal(size=(100, 3))
    assert np.allclose(L.bfr(y, y), 100.0)
    assert np.allclose(L.bfr(y, np.tile(y.mean(0), (100, 1))), 0.0, atol=1e-12)
    z = np.tile(np.array([0.0, 1.0]), 50)[:, None] * np.ones((1, 3))
    assert np.allclose(L.bfr(z, np.zeros_like(z)), (1.0 - np.sqrt(2.0)) * 100.0)


def test_gradient_regularization_exact_and_step_convergence():
    th = L.pack(_theta(10))
    S, K = 2, 15
    # u = 0, x0 = 0: y^ = 0 for every theta, so J = 0 around the point and grad = (s2 th, sx x0)
    us = [np.zeros((K, 3))] * S
    ys = [np.zeros((K, 3))] * S
    x0 = np.zeros((S, 4))
    g = L.gradient_fd(th, x0, us, ys, sigma2=1e-2, sigmax=1e-3)
    assert np.allclose(g[:th.size], 1e-2 * th, rtol=1e-7, atol=1e-10)   # FD rounding ~1e-11
    assert np.allclose(g[th.size:], 0.0, atol=1e-10)
    # generic point: central differences at h and 2h agree
    r = _rng(11)
    us = [r.normal(size=(K, 3)) for _ in range(S)]
    ys = [r.normal(size=(K, 3)) for _ in range(S)]
    x0 = r.normal(size=(S, 4))
    g1 = L.gradient_fd(th, x0, us, ys, h=1e-6)
    g2 = L.gradient_fd(th, x0, us, ys, h=2e-6)
    assert np.abs(g1 - g2).max() <= 1e-6 * np.abs(g1).max()


def test_augment_is_cumulative_sum():
    yh = _rng(12).normal(size=(40, 3))
    xe = L.augment_outputs(yh, 0.05, xe0=np.array([1.0, -2.0, 0.5]))
    ref = np.vstack([np.zeros(3), np.cumsum(yh, 0)[:-1]]) * 0.05 + np.array([1.0, -2.0, 0.5])
    assert np.allclose(xe, ref, rtol=1e-13, atol=1e-13)
    assert np.allclose(L.augment_outputs(np.zeros((5, 3)), 0.05), 0.0)
