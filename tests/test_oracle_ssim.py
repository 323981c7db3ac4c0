"""Pins of the oracle's L1 + D-SSIM loss (NEXT-1, reading R12) against
facts other than its own code: special cases with closed forms, the maximum at x = y,
symmetry, bounds, the SPEC example, and central finite differences of the gradient."""
import math

import numpy as np
import pytest

import oracle

C1, C2 = 0.01 ** 2, 0.03 ** 2


def _mass_1d(n):
    """Fraction of the normalised 11-tap Gaussian (sigma 1.5) that falls inside [0, n) for
    each centre: the window mass seen through zero padding along one axis."""
    g = np.array([math.exp(-(k - 5) ** 2 / (2 * 1.5 ** 2)) for k in range(11)])
    g /= g.sum()
    return np.array([sum(g[k] for k in range(11) if 0 <= i + k - 5 < n) for i in range(n)])


def test_constant_images_closed_form():
    # x = a, y = b everywhere: every window statistic is the constant times the in-image
    # window mass m (separable: m = M(px) M(py)), so with sx^2 = a^2 m (1 - m), sxy = ab m (1-m):
    #   S = (2ab m^2 + C1)(2ab m(1-m) + C2) / (((a^2+b^2) m^2 + C1)((a^2+b^2) m(1-m) + C2))
    H, W, a, b = 13, 17, 0.7, 0.3
    m = np.outer(_mass_1d(H), _mass_1d(W))
    S = (2 * a * b * m * m + C1) * (2 * a * b * m * (1 - m) + C2) / (
        ((a * a + b * b) * m * m + C1) * ((a * a + b * b) * m * (1 - m) + C2))
    x = np.full((H, W, 3), a)
    y = np.full((H, W, 3), b)
    loss, s, _ = oracle.ssim_loss(x, y, lam=1.0)
    assert abs(s - S.mean()) < 1e-13
    assert abs(loss - (1 - S.mean())) < 1e-13
    # a centre whose whole window lies inside (m = 1) reduces to the textbook luminance term
    assert abs(m[6, 8] - 1.0) < 1e-15  # (1 - m ~ 1e-16 is amplified by 1/C2 below)
    assert abs(S[6, 8] - (2 * a * b + C1) / (a * a + b * b + C1)) < 1e-12


def test_identical_images_maximum():
    rng = np.random.default_rng(1)
    x = rng.random((19, 23, 3))
    loss, s, g = oracle.ssim_loss(x, x)
    assert abs(s - 1.0) < 1e-12 and abs(loss) < 1e-12
    assert np.abs(g).max() < 1e-12  # S is maximal at x = y and sign(0) = 0


def test_symmetry_bounds_and_lambda():
    rng = np.random.default_rng(2)
    x, y = rng.random((16, 21, 3)), rng.random((16, 21, 3))
    _, s_xy, _ = oracle.ssim_loss(x, y)
    _, s_yx, _ = oracle.ssim_loss(y, x)
    assert abs(s_xy - s_yx) < 1e-14 and -1.0 <= s_xy <= 1.0
    l0, _, _ = oracle.ssim_loss(x, y, lam=0.0)
    assert abs(l0 - np.abs(x - y).mean()) < 1e-14  # lambda = 0: the L1 of O13
    l1, s1, _ = oracle.ssim_loss(x, y, lam=1.0)
    assert abs(l1 - (1.0 - s1)) < 1e-15


def test_spec_checkerboard_negative():
    # rendered = 1 - target on a binary checkerboard -> SSIM < 0
    yy, xx = np.mgrid[0:24, 0:24]
    t = ((xx + yy) % 2).astype(np.float64)[:, :, None].repeat(3, 2)
    _, s, _ = oracle.ssim_loss(1.0 - t, t)
    assert s < 0.0


def test_gradient_finite_differences():
    rng = np.random.default_rng(3)
    H, W = 14, 15
    x, y = rng.random((H, W, 3)), rng.random((H, W, 3))
    # keep probes away from the L1 kink
    y = np.where(np.abs(x - y) < 0.05, np.clip(x + 0.3, 0, 1), y)
    _, _, g = oracle.ssim_loss(x, y)
    h = 1e-6
    probes = [(int(rng.integers(H)), int(rng.integers(W)), int(rng.integers(3))) for _ in range(60)]
    probes += [(0, 0, 0), (H - 1, W - 1, 2), (0, W - 1, 1), (5, 0, 0)]  # borders (zero padding)
    for (i, j, c) in probes:
        xp, xm = x.copy(), x.copy()
        xp[i, j, c] += h
        xm[i, j, c] -= h
        fd = (oracle.ssim_loss(xp, y, want_grad=False)[0] - oracle.ssim_loss(xm, y, want_grad=False)[0]) / (2 * h)
        assert abs(fd - g[i, j, c]) <= 1e-6 * max(abs(fd), 1e-4), ((i, j, c), fd, g[i, j, c])


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_batch_is_mean_of_images(lam):
    rng = np.random.default_rng(4)
    xs, ys = rng.random((3, 12, 13, 3)), rng.random((3, 12, 13, 3))
    tot, g = oracle.ssim_loss_batch(xs, ys, lam)
    each = [oracle.ssim_loss(xs[i], ys[i], lam) for i in range(3)]
    assert abs(tot - sum(e[0] for e in each) / 3) < 1e-15
    np.testing.assert_allclose(g[1], each[1][2] / 3, rtol=0, atol=1e-18)
