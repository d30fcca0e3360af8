"""Pins of the oracle's kernel functions against mathematics the paper fixes (not against
the oracle's own formulas).  P:n = PAPER.md line n."""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate

import oracle as O
import sph_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("h", [9.42e-3, 2.355e-3, 1.0])
def test_cubic_normalised_in_2d(h):
    """Eq. normkernel P:127-131 and P:275 ("both kernels ... are normalized for x in R^2"):
    int_{R^2} W dA = int_0^inf W(r) 2 pi r dr = 1.  Pins the constant (reading A1) and the
    two polynomial pieces (a dropped piece or wrong power changes the integral)."""
    sp = si.preset(1.0, h=h)
    f = lambda r: O.W_cb(sp, r) * 2.0 * math.pi * r
    val = integrate.quad(f, 0, h, epsabs=0, epsrel=1e-13)[0] + \
        integrate.quad(f, h, 2 * h, epsabs=0, epsrel=1e-13)[0]
    assert abs(val - 1.0) < 1e-12


def test_printed_cubic_constant_integrates_to_three():
    """Reading A1: the printed 15/(14 pi h^2) gives integral exactly 3."""
    sp = si.preset(1.0, w_cb_const=si.W_CB_CONST_PRINTED)
    f = lambda r: O.W_cb(sp, r) * 2.0 * math.pi * r
    val = integrate.quad(f, 0, sp.h)[0] + integrate.quad(f, sp.h, 2 * sp.h)[0]
    assert abs(val - 3.0) < 1e-10


@pytest.mark.parametrize("h", [9.42e-3, 1.0])
def test_spiky_normalised_in_2d(h):
    """Eq. spiky3 P:272-274 + P:275: int (10/(pi h^5)) (h-r)^3 2 pi r dr = 1."""
    sp = si.preset(1.0, h=h)
    val = integrate.quad(lambda r: O.W_s3(sp, r) * 2 * math.pi * r, 0, h, epsabs=0, epsrel=1e-13)[0]
    assert abs(val - 1.0) < 1e-12


def test_kernel_values_at_origin_and_support():
    """Closed forms: W_cb(0) = C*4/h^2 = 10/(7 pi h^2) (q=0: 2^3 - 4*1^3 = 4), W_s3(0) = 10/(pi h^2);
    both vanish at their support (2h resp. h).  Golden numbers from SURVEY 8(c)."""
    g = json.load(open(os.path.join(GOLD, "g1_two_fluid.json")))
    sp = si.preset(1.0)
    h = sp.h
    assert O.W_cb(sp, 0.0) == pytest.approx(10.0 / (7.0 * math.pi * h * h), rel=1e-15)
    assert O.W_s3(sp, 0.0) == pytest.approx(10.0 / (math.pi * h * h), rel=1e-15)
    assert O.W_cb(sp, 0.0) == pytest.approx(g["W_cb_0"], rel=1e-11)
    assert O.W_s3(sp, 0.0) == pytest.approx(g["W_s3_0"], rel=1e-11)
    for r in (2 * h, 2.5 * h, 10 * h):
        assert O.W_cb(sp, r) == 0.0 and O.dW_cb(sp, r) == 0.0
    for r in (h, 1.5 * h):
        assert O.W_s3(sp, r) == 0.0
    assert O.dW_s3(sp, 1.5 * h) == 0.0


@pytest.mark.parametrize("r_over_h", [0.05, 0.3, 0.7, 0.99, 1.01, 1.4, 1.9])
def test_gradient_matches_central_difference(r_over_h):
    """dW/dr (used in nabla_i W_ij) vs a central finite difference of W itself."""
    sp = si.preset(1.0)
    h = sp.h
    r = r_over_h * h
    d = 1e-6 * h
    fd = (O.W_cb(sp, r + d) - O.W_cb(sp, r - d)) / (2 * d)
    assert O.dW_cb(sp, r) == pytest.approx(fd, rel=1e-6)
    if r_over_h < 0.99:
        fd = (O.W_s3(sp, r + d) - O.W_s3(sp, r - d)) / (2 * d)
        assert O.dW_s3(sp, r) == pytest.approx(fd, rel=1e-6)


def test_vector_gradient_fd_spec_point():
    """S:57 example: component-wise central FD of W at r = (0.005, 0.003), h = 9.42 mm."""
    sp = si.preset(1.0)
    rv = np.array([0.005, 0.003])
    r = np.linalg.norm(rv)
    g = O.dW_cb(sp, r) * rv / r
    d = 1e-9
    for c in range(2):
        e = np.zeros(2)
        e[c] = d
        fd = (O.W_cb(sp, np.linalg.norm(rv + e)) - O.W_cb(sp, np.linalg.norm(rv - e))) / (2 * d)
        assert g[c] == pytest.approx(fd, rel=1e-6)


def test_cubic_C1_at_q_equal_1():
    """Both branches meet with equal value and slope at q = 1: W' = -3 C/h^3 (SURVEY 8(c) pin)."""
    sp = si.preset(1.0)
    h = sp.h
    a, b = h * (1 - 1e-12), h * (1 + 1e-12)
    assert O.W_cb(sp, a) == pytest.approx(O.W_cb(sp, b), rel=1e-9)
    assert O.dW_cb(sp, h) == pytest.approx(-3.0 * sp.w_cb_const / h ** 3, rel=1e-14)
    assert O.dW_cb(sp, b) == pytest.approx(-3.0 * sp.w_cb_const / h ** 3, rel=1e-9)
    assert O.dW_cb(sp, 0.0) == 0.0  # smooth peak at the origin
