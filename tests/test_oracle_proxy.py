"""Pins for oracle.proxy, x_tilde = Phi^T y -- CPU only."""
import math

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


# ----------------------------------------------------------------------------- sensing model (NEXT-1)
def test_measure_vs_numpy_loop_and_adjoint():
    """y = Phi x: numpy matmul, an explicit loop on a tiny case, and the adjoint identity
    <Phi x, y> = <x, Phi^T y> against the (independently pinned) proxy."""
    r = np.random.default_rng(3)
    phi = r.standard_normal((7, 12))
    x = r.standard_normal((3, 3, 4))
    y = oracle.measure(phi, x)
    assert np.allclose(y, x.reshape(3, 12) @ phi.T, rtol=1e-13, atol=1e-13)
    loop = [[sum(phi[i][j] * x.reshape(3, 12)[b][j] for j in range(12)) for i in range(7)] for b in range(3)]
    assert np.allclose(y, np.array(loop), rtol=1e-13, atol=1e-13)
    w = r.standard_normal((3, 7))
    lhs = np.sum(y * w, axis=1)
    rhs = np.sum(x.reshape(3, 12) * oracle.proxy(phi, w), axis=1)
    assert np.allclose(lhs, rhs, rtol=1e-12)


def test_measure_identity_and_zero():
    x = np.arange(16, dtype=np.float64).reshape(1, 4, 4)
    assert np.array_equal(oracle.measure(np.eye(16), x), x.reshape(1, 16))
    assert np.all(oracle.measure(np.ones((3, 16)), np.zeros((2, 16))) == 0)


def test_noise_snr_rule_determinism_and_noiseless():
    """+inf -> unchanged; 20 dB -> mean ||w||^2/||y||^2 within [0.005, 0.02] over 100 draws;
    same seed -> identical vector."""
    r = np.random.default_rng(5)
    y = r.standard_normal((100, 410))
    assert np.array_equal(oracle.add_noise(y, math.inf, 1), y)
    ratios = [np.sum((oracle.add_noise(y[i:i + 1], 20.0, 7 + i) - y[i:i + 1]) ** 2) / np.sum(y[i] ** 2)
              for i in range(100)]
    assert 0.005 <= float(np.mean(ratios)) <= 0.02
    assert abs(float(np.mean(ratios)) - 0.01) < 0.001    # 100 x 410 samples: tight around the target
    assert np.array_equal(oracle.add_noise(y[:3], 20.0, 11), oracle.add_noise(y[:3], 20.0, 11))
    assert not np.array_equal(oracle.add_noise(y[:3], 20.0, 11), oracle.add_noise(y[:3], 20.0, 12))
    with pytest.raises(ValueError):
        oracle.add_noise(np.zeros((1, 4)), 20.0, 1)
