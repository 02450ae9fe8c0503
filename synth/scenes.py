"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no projection, covariance, SH
evaluation, compositing or gradients).  It only draws parameters: Gaussian means,
quaternions, activated scales and opacities, SH coefficients, camera poses and
intrinsics, and upstream image gradients.  Recipes are SURVEY.md section 8(d) and
are restated in DESIGN.md "Input recipe".

All arrays are float32 (the dtype the C-ABI takes) except where noted.  A scene is
a plain dict:
  means [N,3], quats [N,4] (w,x,y,z, unnormalised), scales [N,3] (activated, >0),
  opacities [N] (activated, in (0,1)), colors [N,K,3] (SH) or [N,3] (direct RGB),
  sh_degree (int, -1 for direct RGB), viewmats [C,4,4] (world->camera, OpenCV axes),
  Ks [C,3,3], width, height.
"""
from __future__ import annotations

import numpy as np

# Config names follow BASELINE.json "configs" (index 0..4).
CONFIGS = {
    "tiny": dict(N=100, width=64, height=64, views=1, sh_degree=0, seed=0),                # configs[0]
    "garden1m": dict(N=1_000_000, width=1297, height=840, views=1, sh_degree=3, seed=1002),  # configs[1]
    "batch3m": dict(N=3_000_000, width=1297, height=840, views=8, sh_degree=3, seed=1003),   # configs[2]
    "large6m": dict(N=6_000_000, width=1920, height=1080, views=32, sh_degree=3, seed=1004),  # configs[3]
    "aa_packed1m": dict(N=1_000_000, width=1297, height=840, views=4, sh_degree=3, seed=1005,
                        antialiased=1, packed=1),                                              # configs[4]
}


def _lookat_viewmat(pos, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0)):
    """World->camera matrix for a camera at `pos` looking at `target`; OpenCV axes
    (x right, y down, z forward).  Input construction only."""
    pos = np.asarray(pos, np.float64)
    f = np.asarray(target, np.float64) - pos
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f])          # rows: camera axes in world coordinates
    V = np.eye(4)
    V[:3, :3] = R
    V[:3, 3] = -R @ pos
    return V


def intrinsics(width, height, focal_frac=0.85):
    f = focal_frac * width
    return np.array([[f, 0.0, width / 2.0], [0.0, f, height / 2.0], [0.0, 0.0, 1.0]])


def orbit_cameras(n_views, width, height, seed, radius=3.2, view_offset=0):
    """Look-at-origin cameras on an orbit: azimuth evenly spaced by view index,
    elevation U(10, 35) degrees, fx = fy = 0.85 W, principal point at the centre."""
    rng = np.random.default_rng(seed + 7919)
    total = max(n_views + view_offset, 1)
    elev = rng.uniform(10.0, 35.0, size=total)
    viewmats, Ks = [], []
    for v in range(view_offset, view_offset + n_views):
        az = 2.0 * np.pi * v / 8.0
        el = np.deg2rad(elev[v])
        pos = radius * np.array([np.cos(el) * np.sin(az), np.sin(el), -np.cos(el) * np.cos(az)])
        viewmats.append(_lookat_viewmat(pos))
        Ks.append(intrinsics(width, height))
    return np.asarray(viewmats, np.float32), np.asarray(Ks, np.float32)


def _random_sh(rng, N, sh_degree, dc_std=0.6, band_std=(0.05, 0.03, 0.02)):
    if sh_degree < 0:
        return rng.uniform(0.0, 1.0, size=(N, 3)).astype(np.float32)
    K = (sh_degree + 1) ** 2
    sh = np.zeros((N, K, 3), np.float32)
    sh[:, 0, :] = rng.normal(0.0, dc_std, size=(N, 3))
    lo = 1
    for band in range(1, sh_degree + 1):
        hi = (band + 1) ** 2
        sh[:, lo:hi, :] = rng.normal(0.0, band_std[band - 1], size=(N, hi - lo, 3))
        lo = hi
    return sh


def _quat_mul(a, b):
    """Hamilton product of (w,x,y,z) quaternions, row-wise (input construction only)."""
    w1, x1, y1, z1 = a.T
    w2, x2, y2, z2 = b.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=1)


def _quats_aligned(rng, normals):
    """Quaternions whose local z axis maps to `normals` (thin axis = scale[2]), with a
    uniformly random spin about that axis."""
    n = normals / np.linalg.norm(normals, axis=1, keepdims=True)
    # shortest arc z -> n : q = normalise(1 + n_z, -n_y, n_x, 0); guard n = -z
    q = np.stack([1.0 + n[:, 2], -n[:, 1], n[:, 0], np.zeros(len(n))], axis=1)
    bad = q[:, 0] < 1e-6
    q[bad] = np.array([0.0, 1.0, 0.0, 0.0])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    phi = rng.uniform(0, 2 * np.pi, size=len(n))
    spin = np.stack([np.cos(phi / 2), np.zeros_like(phi), np.zeros_like(phi), np.sin(phi / 2)], axis=1)
    return _quat_mul(q, spin)


def mipnerf_like_scene(N, width=1297, height=840, views=1, sh_degree=3, seed=1002, view_offset=0):
    """SURVEY 8(d) "MipNeRF360-like" generator: 45 % on a noisy central object (sphere /
    torus mix, radius ~1), 25 % on a ground disk (radius 3, y = -1), 30 % in a
    background shell r in [4, 20] with density ~ r^-2; surface-aligned anisotropic
    scales; bimodal opacities; SH with decaying band energy; orbit cameras."""
    rng = np.random.default_rng(seed)
    n_obj = int(0.45 * N)
    n_gnd = int(0.25 * N)
    n_bg = N - n_obj - n_gnd
    n_sph = n_obj // 2
    n_tor = n_obj - n_sph

    # sphere radius 1 centred at origin
    d = rng.normal(size=(n_sph, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p_sph = d * (1.0 + rng.normal(0, 0.02, size=(n_sph, 1)))
    nrm_sph = d
    # torus around the sphere: major R = 1.3, minor r = 0.25, lying in the xz plane
    u = rng.uniform(0, 2 * np.pi, n_tor)
    v = rng.uniform(0, 2 * np.pi, n_tor)
    Rt, rt = 1.3, 0.25
    cen = np.stack([Rt * np.cos(u), np.zeros(n_tor), Rt * np.sin(u)], axis=1)
    nrm_tor = np.stack([np.cos(v) * np.cos(u), np.sin(v), np.cos(v) * np.sin(u)], axis=1)
    p_tor = cen + (rt + rng.normal(0, 0.01, size=(n_tor, 1))) * nrm_tor
    area_obj = 4 * np.pi * 1.0 + 4 * np.pi ** 2 * Rt * rt
    # ground disk radius 3 at y = -1
    rr = 3.0 * np.sqrt(rng.uniform(0, 1, n_gnd))
    th = rng.uniform(0, 2 * np.pi, n_gnd)
    p_gnd = np.stack([rr * np.cos(th), -1.0 + rng.normal(0, 0.01, n_gnd), rr * np.sin(th)], axis=1)
    nrm_gnd = np.tile(np.array([[0.0, 1.0, 0.0]]), (n_gnd, 1))
    area_gnd = np.pi * 9.0
    # background shell: radial pdf uniform on [4, 20] (volume density ~ r^-2), upper-biased
    rb = rng.uniform(4.0, 20.0, n_bg)
    db = rng.normal(size=(n_bg, 3))
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    db[:, 1] = np.abs(db[:, 1]) * 0.8 - 0.1
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    p_bg = db * rb[:, None]

    means = np.concatenate([p_sph, p_tor, p_gnd, p_bg]).astype(np.float32)

    sp_obj = np.sqrt(area_obj / max(n_obj, 1))
    sp_gnd = np.sqrt(area_gnd / max(n_gnd, 1))
    def surf_scales(n, spacing):
        t = spacing * rng.lognormal(0.0, 0.4, size=(n, 2))
        return np.concatenate([t, 0.15 * t.min(axis=1, keepdims=True)], axis=1)
    s_obj = surf_scales(n_obj, sp_obj)
    s_gnd = surf_scales(n_gnd, sp_gnd)
    s_bg = 0.01 * rb[:, None] * rng.lognormal(0.0, 0.5, size=(n_bg, 3))
    scales = np.concatenate([s_obj, s_gnd, s_bg]).astype(np.float32)

    q_obj = _quats_aligned(rng, np.concatenate([nrm_sph, nrm_tor]))
    q_gnd = _quats_aligned(rng, nrm_gnd)
    q_bg = rng.normal(size=(n_bg, 4))
    quats = np.concatenate([q_obj, q_gnd, q_bg]).astype(np.float32)
    # unnormalised on input (the method normalises, F1): random positive rescale
    quats *= rng.uniform(0.5, 2.0, size=(N, 1)).astype(np.float32)

    mode = rng.uniform(size=N) < 0.5
    opac = np.where(mode, rng.beta(0.6, 3.0, N), rng.beta(6.0, 1.0, N))
    opac = np.clip(opac, 1e-3, 1 - 1e-3).astype(np.float32)

    perm = rng.permutation(N)   # interleave regions in memory like a trained model
    colors = _random_sh(rng, N, sh_degree)
    viewmats, Ks = orbit_cameras(views, width, height, seed, view_offset=view_offset)
    return dict(means=means[perm], quats=quats[perm], scales=scales[perm], opacities=opac[perm],
                colors=colors, sh_degree=sh_degree, viewmats=viewmats, Ks=Ks,
                width=width, height=height)


def tiny_scene(seed=0, N=100, width=64, height=64, sh_degree=0, views=1):
    """BASELINE configs[0] recipe: identity view, f = 64, c = 32,
    z ~ U(2,6), x,y ~ U(-0.45 z, 0.45 z), log-uniform scales in [0.03, 0.3],
    quats ~ N(0, I4) unnormalised, opacities U(0.05, 0.95), SH dc ~ N(0, 1)."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(2.0, 6.0, N)
    x = rng.uniform(-0.45, 0.45, N) * z
    y = rng.uniform(-0.45, 0.45, N) * z
    means = np.stack([x, y, z], axis=1).astype(np.float32)
    scales = np.exp(rng.uniform(np.log(0.03), np.log(0.3), size=(N, 3))).astype(np.float32)
    quats = rng.normal(size=(N, 4)).astype(np.float32)
    opac = rng.uniform(0.05, 0.95, N).astype(np.float32)
    if sh_degree < 0:
        colors = rng.uniform(0, 1, size=(N, 3)).astype(np.float32)
    else:
        K = (sh_degree + 1) ** 2
        colors = np.zeros((N, K, 3), np.float32)
        colors[:, 0, :] = rng.normal(0, 1, size=(N, 3))
        if K > 1:
            colors[:, 1:, :] = rng.normal(0, 0.3, size=(N, K - 1, 3))
    f = 64.0 * width / 64.0
    viewmats = np.tile(np.eye(4, dtype=np.float32), (views, 1, 1))
    if views > 1:
        # small sideways translations for extra views (input construction only)
        viewmats[:, 0, 3] = np.linspace(-0.2, 0.2, views)
    Ks = np.tile(np.array([[f, 0, width / 2.0], [0, f, height / 2.0], [0, 0, 1]], np.float32), (views, 1, 1))
    return dict(means=means, quats=quats, scales=scales, opacities=opac, colors=colors,
                sh_degree=sh_degree, viewmats=viewmats, Ks=Ks, width=width, height=height)


def fig1_scene(scale=(0.5, 0.5, 0.5), color=(0.2, 0.6, 0.9)):
    """The paper's Fig. 1: one Gaussian at (0,0,0.01), identity quaternion,
    opacity 1, identity view, K = [[1,0,120],[0,1,120],[0,0,1]], 240 x 240, direct RGB.
    (`torch.rand` scale/colour are fixed to given values here.)"""
    return dict(means=np.array([[0.0, 0.0, 0.01]], np.float32),
                quats=np.array([[1.0, 0.0, 0.0, 0.0]], np.float32),
                scales=np.array([scale], np.float32), opacities=np.array([1.0], np.float32),
                colors=np.array([color], np.float32), sh_degree=-1,
                viewmats=np.eye(4, dtype=np.float32)[None],
                Ks=np.array([[[1.0, 0.0, 120.0], [0.0, 1.0, 120.0], [0.0, 0.0, 1.0]]], np.float32),
                width=240, height=240)


def image_grads(seed, C, H, W, l1_scale=True, with_alpha=False):
    """Upstream dL/d(image): N(0, (1/(3HW))^2) -- the scale of an L1 loss gradient
     -- or N(0,1) when l1_scale is False (small parity cases)."""
    rng = np.random.default_rng(seed + 104729)
    sd = 1.0 / (3.0 * H * W) if l1_scale else 1.0
    v = rng.normal(0.0, sd, size=(C, H, W, 3)).astype(np.float32)
    va = rng.normal(0.0, sd, size=(C, H, W)).astype(np.float32) if with_alpha else None
    return v, va


def tile_subset_mask(seed, C, W, H, n_tiles, tile=16):
    """Seeded subset of tiles per view (for masked-loss parity / oracle timing at scale)."""
    rng = np.random.default_rng(seed + 15485863)
    TX, TY = (W + tile - 1) // tile, (H + tile - 1) // tile
    mask = np.zeros((C, TY * TX), np.uint8)
    for c in range(C):
        sel = rng.choice(TY * TX, size=min(n_tiles, TY * TX), replace=False)
        mask[c, sel] = 1
    return mask.reshape(C, TY, TX)


def scene_from_config(name, views=None, N=None, view_offset=0):
    cfg = dict(CONFIGS[name])
    if N is not None:
        cfg["N"] = N
    if views is not None:
        cfg["views"] = views
    if name == "tiny":
        return tiny_scene(seed=cfg["seed"], N=cfg["N"], width=cfg["width"], height=cfg["height"],
                          sh_degree=cfg["sh_degree"], views=cfg["views"])
    return mipnerf_like_scene(cfg["N"], cfg["width"], cfg["height"], cfg["views"], cfg["sh_degree"],
                              cfg["seed"], view_offset=view_offset)
