"""Pins for the oracle's handling of ambiguous threshold decisions (DESIGN Q28b): a decision
that lies within the fp32 error bound admits both outcomes, the oracle enumerates them
(flip masks) and bounds the gradient difference they make.  Closed forms on hand-built
splats; CPU only."""
import math

import numpy as np

import oracle
from synth import scenes as S
from tests.test_oracle_pins import _splat2d

AMIN = 1.0 / 255.0


def _one_splat(opac, dx=0.25, var=4.0, rgb=(0.2, 0.6, 0.9)):
    """One isotropic splat of variance var px^2 centred dx px right of pixel (8, 8)'s centre."""
    A = 1.0 / var
    return _splat2d([[8.5 + dx, 8.5]], [[A, 0.0, A]], [opac], [list(rgb)], [2.0], [[6, 6]]), 0.5 * A * dx * dx


def test_flip_of_an_ambiguous_alpha_min_decision_is_the_other_outcome():
    """alpha = o e^-sigma within a few ulp of alpha_min at pixel (8, 8) (Q14): the
    pixel is flagged; outcome 0 is the fp64 decision, outcome 1 the other one, each equal to
    its closed form -- composited (T = 1 - alpha, C = c alpha) or skipped (T = 1, C = 0)."""
    sigma = 0.5 * 0.25 * 0.0625
    o32 = float(np.float32(AMIN * math.exp(sigma)))
    p, sigma = _one_splat(o32)
    opts = oracle.Options(sh_degree=-1)
    f = oracle.render_fwd(p, 1, 1, 16, 16, opts)
    assert f["ambig"][0, 8, 8] == 1
    assert f["ambig"].sum() == 1                       # every other pixel is far from a threshold
    alpha = o32 * math.exp(-sigma)
    took = alpha >= AMIN
    r = oracle.render_pixels(p, 1, 1, 16, 16, opts, [0, 0], [8, 8], [8, 8], [0, 1])
    for q, inc in ((0, took), (1, not took)):
        if inc:
            assert math.isclose(r["T"][q], 1 - alpha, rel_tol=1e-14)
            assert np.allclose(r["rgb"][q], np.array([0.2, 0.6, 0.9]) * alpha, rtol=1e-14, atol=0)
            assert r["last_gid"][q] == 0
        else:
            assert r["T"][q] == 1.0 and np.all(r["rgb"][q] == 0) and r["last_gid"][q] == -1
    assert np.array_equal(r["namb"], [1, 1])
    # flips through render_fwd agree with the single-pixel evaluation
    fl = np.zeros((1, 16, 16), np.uint32)
    fl[0, 8, 8] = 1
    f1 = oracle.render_fwd(p, 1, 1, 16, 16, opts, flips=fl)
    assert f1["T"][0, 8, 8] == r["T"][1] and np.array_equal(f1["rgb"][0, 8, 8], r["rgb"][1])
    other = np.ones((16, 16), bool)
    other[8, 8] = False
    assert np.array_equal(f1["rgb"][0][other], f["rgb"][0][other])


def test_d2d_is_the_gradient_difference_of_an_ambiguous_saturation():
    """o e^-sigma within a few ulp of alpha_max = 0.99 (Q13): B6 gives no sigma / opacity
    gradient when saturated and the full one when not (Q24).  The oracle's d2d at that splat
    equals |v2d(outcome 1) - v2d(outcome 0)| (slots mean2d, conic, opacity), and 0 elsewhere."""
    sigma = 0.5 * 0.25 * 0.0625
    o32 = float(np.float32(0.99 * math.exp(sigma)))
    p, _ = _one_splat(o32)
    opts = oracle.Options(sh_degree=-1)
    f = oracle.render_fwd(p, 1, 1, 16, 16, opts)
    assert f["ambig"][0, 8, 8] == 1 and f["ambig"].sum() == 1
    v = np.zeros((1, 16, 16, 3))
    v[0, 8, 8] = (0.3, -0.7, 0.4)
    fl = np.zeros((1, 16, 16), np.uint32)
    fl[0, 8, 8] = 1
    b0 = oracle.render_bwd(p, 1, 1, 16, 16, opts, v)
    b1 = oracle.render_bwd(p, 1, 1, 16, 16, opts, v, flips=fl)
    diff = np.abs(b1["v2d"] - b0["v2d"])[0, 0]
    d = b0["d2d"][0, 0]
    for j in (0, 1, 2, 3, 4, 8):   # oracle layout: mean2d 0-1, conic 2-4, rgb 5-7, opacity 8
        assert math.isclose(diff[j], d[j], rel_tol=1e-5), (j, diff[j], d[j])
    assert d[8] > 0 and np.all(d[5:8] == 0)
    # a pixel with no ambiguous decision contributes nothing to d2d
    v2 = np.zeros_like(v)
    v2[0, 8, 10] = 1.0
    assert np.all(oracle.render_bwd(p, 1, 1, 16, 16, opts, v2)["d2d"] == 0)


def test_sh_clamp_alternative_is_the_unclamped_colour_path():
    """colour = max(0, 0.5 + Y0 dc) (Q22) with 0.5 + Y0 dc within the fp32 rounding of 0:
    both clamp outcomes are correct; project_bwd_clamp_alt gives |Y0 v_rgb| on that channel's
    dc coefficient (SH degree 0: no view-direction term) and 0 on the clearly unclamped ones."""
    Y0 = 0.28209479177387814
    dc = np.float32(-0.5 / Y0)
    sc = dict(means=np.array([[0.0, 0.0, 3.0]], np.float32), quats=np.array([[1, 0, 0, 0]], np.float32),
              scales=np.array([[0.1, 0.1, 0.1]], np.float32), opacities=np.array([0.5], np.float32),
              colors=np.array([[[dc, 1.0, -3.0]]], np.float32), sh_degree=0,
              viewmats=np.eye(4, dtype=np.float32)[None],
              Ks=np.array([[[64, 0, 32], [0, 64, 32], [0, 0, 1]]], np.float32), width=64, height=64)
    opts = oracle.Options(sh_degree=0)
    p = oracle.project(sc, opts)
    assert abs(0.5 + Y0 * float(dc)) < 1e-7
    v2d = np.zeros((1, 1, 9))
    v2d[0, 0, 5:8] = (0.7, -0.2, 0.9)
    alt = oracle.project_bwd_clamp_alt(sc, p, v2d, opts)
    assert math.isclose(alt["v_colors"][0, 0, 0], Y0 * 0.7, rel_tol=1e-12)
    assert alt["v_colors"][0, 0, 1] == 0 and alt["v_colors"][0, 0, 2] == 0
    assert np.all(alt["v_means"] == 0) and np.all(alt["v_quats"] == 0)


def test_render_pixels_without_flips_equals_render_fwd():
    sc = S.mipnerf_like_scene(3000, width=96, height=64, views=2, sh_degree=3, seed=5)
    opts = oracle.Options(sh_degree=3)
    p = oracle.project(sc, opts)
    f = oracle.render_fwd(p, 2, 3000, 96, 64, opts)
    rng = np.random.default_rng(0)
    cams, ys, xs = rng.integers(0, 2, 200), rng.integers(0, 64, 200), rng.integers(0, 96, 200)
    r = oracle.render_pixels(p, 2, 3000, 96, 64, opts, cams, xs, ys, np.zeros(200, np.uint32))
    assert np.array_equal(r["rgb"], f["rgb"][cams, ys, xs])
    assert np.array_equal(r["T"], f["T"][cams, ys, xs])
    assert np.array_equal(r["last_gid"], f["last_gid"][cams, ys, xs])
    assert np.array_equal(r["namb"], f["ambig"][cams, ys, xs])
