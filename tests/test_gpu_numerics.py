"""Pins of the renderer's error model (DESIGN.md §2 R16) on the device it runs on: the
constant part of the oracle's alpha error bound (oracle.MARGINS alpha_abs) must cover the
measured relative error of ex2.approx (the alpha = o 2^-q of A4/A5) plus the roundings of
the opacity and of the product o G (2 u_r)."""
import pytest

import oracle

L = pytest.importorskip("paper_2406_18533_b200._lib")
pytestmark = pytest.mark.gpu


def test_ex2_error_within_alpha_margin():
    ctx = L.Context(0, 0, 1)
    # every fp32 exponent a composited or skipped alpha can take: q in [0, 60] (alpha >= 1/255
    # needs q <= log2(255) < 8; larger q only matter below the skip threshold)
    err = L.selftest_ex2(ctx, -60.0, 0.0)
    print("ex2.approx.ftz max relative error over [-60, 0]: %.3e (2^%.2f)" % (err, __import__("math").log2(err)))
    assert err + 2 * 2.0 ** -24 <= oracle.MARGINS[3], err
