"""Pins for oracle.proxy, x_tilde = Phi^T y -- CPU only."""
import numpy as np
import pytest

import oracle
import synth

RNG = np.random.default_rng(17)


def test_proxy_vs_numpy_and_triple_loop():
    m, n, b = 7, 12, 3
    phi = RNG.standard_normal((m, n))
    y = RNG.standard_normal((b, m))
    got = oracle.proxy(phi, y)
    np.testing.assert_allclose(got, y @ phi, rtol=0, atol=1e-13)
    loop = np.zeros((b, n))
    for bb in range(b):
        for j in range(n):
            for i in range(m):
                loop[bb, j] += phi[i, j] * y[bb, i]
    np.testing.assert_allclose(got, loop, rtol=0, atol=1e-13)


def test_adjoint_dot_test_over_seeds():
    """<Phi x, y> = <x, Phi^T y> on generated ensembles."""
    for seed in range(20):
        phi = synth.make_phi(40, 96, seed=seed).astype(np.float64)
        x = RNG.standard_normal(96)
        y = RNG.standard_normal(40)
        lhs = float((phi @ x) @ y)
        rhs = float(x @ oracle.proxy(phi, y)[0])
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_identity_phi_reshapes_y():
    n1, n2 = 4, 6
    y = RNG.standard_normal((2, n1 * n2))
    got = oracle.proxy(np.eye(n1 * n2), y)
    assert np.array_equal(got, y)


def test_unit_vector_selects_phi_row():
    """y = e_i gives x_tilde = row i of Phi (laid out row-major, j = r*n2 + c)."""
    phi = RNG.standard_normal((5, 20))
    for i in range(5):
        e = np.zeros(5)
        e[i] = 1.0
        assert np.array_equal(oracle.proxy(phi, e)[0], phi[i])


def test_zero_measurements_give_zero_proxy():
    phi = RNG.standard_normal((5, 20))
    assert np.all(oracle.proxy(phi, np.zeros((3, 5))) == 0)


def test_orthonormal_square_phi_inverts():
    q, _ = np.linalg.qr(RNG.standard_normal((30, 30)))
    x = RNG.standard_normal(30)
    np.testing.assert_allclose(oracle.proxy(q, q @ x)[0], x, rtol=0, atol=1e-12)


def test_proxy_psd_and_linear():
    phi = RNG.standard_normal((10, 25))
    x1, x2 = RNG.standard_normal((2, 25))
    g = lambda v: oracle.proxy(phi, phi @ v)[0]
    assert x1 @ g(x1) >= 0
    np.testing.assert_allclose(g(2 * x1 - x2), 2 * g(x1) - g(x2), rtol=0, atol=1e-11)


def test_bad_shapes_raise():
    with pytest.raises(ValueError):
        oracle.proxy(np.zeros((0, 4)), np.zeros((1, 0)))
