"""Pins of the steering-weight oracle (Eqs. 1-3) against closed forms:
zero offset / broadside -> 1; half-wavelength uniform line -> exp(i pi k sin theta) (textbook
ULA steering vector); mirror symmetry theta -> -theta is the conjugate; and the weights
beamform a simulated far-field plane wave to the Dirichlet response with peak K at the source
angle (coherent gain)."""
import numpy as np

import oracle


def test_broadside_and_reference_element():
    w = oracle.steering_weights([0.0, 1.5, 7.0], [0.0, 0.3], [150e6, 1.0e6], 3e8)
    assert np.allclose(w[:, 0, :], 1.0, atol=0, rtol=0)      # theta = 0: tau = 0
    assert np.allclose(w[:, :, 0], 1.0, atol=0, rtol=0)      # d = 0: tau = 0


def test_half_wavelength_ula_closed_form():
    c, f = 343.0, 1000.0                       # acoustic wave, lambda = 0.343 m
    lam = c / f
    K = 16
    d = np.arange(K) * lam / 2
    th = np.deg2rad([-60.0, -10.0, 0.0, 25.0, 80.0])
    w = oracle.steering_weights(d, th, [f], c)[0]
    expect = np.exp(1j * np.pi * np.outer(np.sin(th), np.arange(K)))
    assert np.max(np.abs(w - expect)) < 1e-12


def test_mirror_angle_is_conjugate():
    d = np.array([0.0, 0.7, 3.1, 12.0])
    w = oracle.steering_weights(d, [0.4, -0.4], [2.0e8], 3e8)[0]
    assert np.max(np.abs(w[1] - np.conj(w[0]))) < 1e-12


def test_coherent_gain_on_simulated_plane_wave():
    """x_k = s exp(-2 pi i f tau_k(theta0)) (Eq. 1 narrowband): |sum_k w_k x_k| peaks at theta0 with
    magnitude K |s| (Eq. 3)."""
    c, f = 3e8, 150e6
    lam = c / f
    K = 48
    rng = np.random.default_rng(3)
    d = np.sort(rng.uniform(0, 20 * lam, K))
    th = np.deg2rad(np.linspace(-70, 70, 141))
    t0 = th[97]
    x = np.exp(-2j * np.pi * f * d * np.sin(t0) / c)
    w = oracle.steering_weights(d, th, [f], c)[0]
    y = w @ x
    assert int(np.argmax(np.abs(y))) == 97
    assert abs(abs(y[97]) - K) < 1e-9
