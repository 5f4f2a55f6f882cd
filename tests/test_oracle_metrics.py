"""Pins for oracle.rel_l2, the parity statistic of BASELINE.json north_star (||a - b||_2 / ||b||_2) -- CPU only.

Closed forms: a vector against itself, its double, its negation and zero; right-angle cases whose norms are
integers (3-4-5); the zero-reference conventions; and invariance under flattening (the statistic is taken over
the whole image, not row by row).  A swapped argument order, a missing square root or a squared norm fails one
of them."""
import math

import numpy as np
import pytest

import oracle


def test_identity_is_zero():
    b = np.random.default_rng(0).standard_normal((7, 9))
    assert oracle.rel_l2(b, b) == 0.0


def test_double_and_negation():
    b = np.random.default_rng(1).standard_normal(33)
    assert oracle.rel_l2(2 * b, b) == pytest.approx(1.0, abs=1e-15)
    assert oracle.rel_l2(-b, b) == pytest.approx(2.0, abs=1e-15)
    assert oracle.rel_l2(np.zeros_like(b), b) == pytest.approx(1.0, abs=1e-15)


def test_integer_norm_cases_and_argument_order():
    # a - b = (3, -4): ||.|| = 5; ||b|| = 4 -> 5/4; swapped: ||a|| = 3 -> 5/3 (order matters)
    a, b = np.array([3.0, 0.0]), np.array([0.0, 4.0])
    assert oracle.rel_l2(a, b) == 1.25
    assert oracle.rel_l2(b, a) == pytest.approx(5.0 / 3.0, abs=1e-15)
    # not squared: a - b = (0, 0, 12), ||b|| = ||(3, 4, 0)|| = 5 -> 12/5
    assert oracle.rel_l2([3.0, 4.0, 12.0], [3.0, 4.0, 0.0]) == pytest.approx(2.4, abs=1e-15)


def test_zero_reference_conventions():
    z = np.zeros(5)
    assert oracle.rel_l2(z, z) == 0.0
    assert oracle.rel_l2(z + 1.0, z) == math.inf


def test_whole_image_not_per_row():
    # rows with different errors: the statistic is over all elements
    b = np.array([[1.0, 0.0], [0.0, 1.0]])
    a = np.array([[1.0, 0.0], [0.0, 3.0]])
    assert oracle.rel_l2(a, b) == pytest.approx(2.0 / math.sqrt(2.0), abs=1e-15)
    assert oracle.rel_l2(a, b) == oracle.rel_l2(a.ravel(), b.ravel())
