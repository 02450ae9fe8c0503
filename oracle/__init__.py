"""CPU oracle for the gsplat hot path (arXiv 2409.06765) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2409_06765_b200`` never imports it, and the two share no code: this
wrapper marshals numpy arrays into ``liboracle`` (``gs_oracle.c``) and nothing
else.  See the header of ``gs_oracle.c`` for what each function follows in the
paper, and DESIGN.md "Oracle pins" for what pins each one.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gs_oracle.c")
_LIB = os.path.join(_HERE, "libgs_oracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile gs_oracle.c (plain C, OpenMP) into oracle/libgs_oracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class OrOpts(ct.Structure):
    _fields_ = [
        ("near_plane", ct.c_double), ("far_plane", ct.c_double), ("eps2d", ct.c_double),
        ("alpha_max", ct.c_double), ("alpha_min", ct.c_double), ("t_min", ct.c_double),
        ("amb_safety", ct.c_double), ("amb_rel_floor", ct.c_double),
        ("tile_size", ct.c_int32), ("antialiased", ct.c_int32), ("sh_degree", ct.c_int32),
        ("bbox_mode", ct.c_int32), ("fov_clamp", ct.c_int32), ("channels", ct.c_int32),
    ]


@dataclass
class Options:
    """Constants of the method.  Duplicated, not shared, with the
    CUDA path's gs_options; tests/test_abi.py cross-checks the two tables."""
    near_plane: float = 0.01       # S:196, Q18
    far_plane: float = 1e10
    eps2d: float = 0.3
    alpha_max: float = 0.99        # north_star "opacity saturation at 0.99" (Q13)
    alpha_min: float = 1.0 / 255.0  # Q14
    t_min: float = 1e-4            # Q15
    amb_safety: float = 1.5        # ambiguity flags (Q28b): factor on the derived fp32
    amb_rel_floor: float = 0.0     #   error bound of each decision; minimum relative margin
    tile_size: int = 16
    antialiased: int = 0
    sh_degree: int = 3
    bbox_mode: int = 0
    channels: int = 0              # 0: RGB from the projection; D > 0: N-D features (render_*_nd)
    fov_clamp: int = 1

    def c(self) -> OrOpts:
        return OrOpts(self.near_plane, self.far_plane, self.eps2d, self.alpha_max, self.alpha_min,
                      self.t_min, self.amb_safety, self.amb_rel_floor, self.tile_size, self.antialiased,
                      self.sh_degree, self.bbox_mode, self.fov_clamp, int(self.channels))


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        P = ct.c_void_p
        i64, i32, dbl = ct.c_int64, ct.c_int32, ct.c_double
        _lib.or_project.argtypes = [P, i64, i32, i32, i32] + [P] * 5 + [i32, P, P] + [P] * 10
        _lib.or_isect.argtypes = [P, i32, i64, i32, i32, P, P, P, i64, P, P, P]
        _lib.or_isect.restype = i64
        _lib.or_render_fwd.argtypes = [P, i32, i64, i32, i32] + [P] * 10 + [P] * 6 + [P] * 2 + [P]
        _lib.or_render_bwd.argtypes = [P, i32, i64, i32, i32] + [P] * 10 + [P] * 7 + [P] * 8 + [P] * 4
        _lib.or_render_pixels.argtypes = [P, i32, i64, i32, i32] + [P] * 9 + [i64] + [P] * 8
        _lib.or_project_bwd.argtypes = [P, i64, i32, i32, i32] + [P] * 5 + [i32] + [P] * 3 + [P] * 6 + [P] * 2 + [i32]
        _lib.or_sh_basis.argtypes = [i32, dbl, dbl, dbl, P]
        _lib.or_sh_basis_grad.argtypes = [i32, dbl, dbl, dbl, P]
        _lib.or_quat_to_rotmat.argtypes = [P, P]
        _lib.or_num_threads.restype = i32
        _lib.or_set_num_threads.argtypes = [i32]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ct.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return lib().or_num_threads()


def set_num_threads(n: int) -> None:
    lib().or_set_num_threads(int(n))


def sh_basis(deg, d):
    Y = np.zeros(16)
    lib().or_sh_basis(deg, float(d[0]), float(d[1]), float(d[2]), _p(Y))
    return Y[: (deg + 1) ** 2]


def sh_basis_grad(deg, d):
    g = np.zeros((16, 3))
    lib().or_sh_basis_grad(deg, float(d[0]), float(d[1]), float(d[2]), _p(g))
    return g[: (deg + 1) ** 2]


def quat_to_rotmat(q):
    R = np.zeros((3, 3))
    lib().or_quat_to_rotmat(_p(_f64(q)), _p(R))
    return R


def _scene_arrays(scene):
    means = _f32(scene["means"]); quats = _f32(scene["quats"]); scales = _f32(scene["scales"])
    opac = _f32(scene["opacities"]); colors = _f32(scene["colors"])
    viewmats = _f32(scene["viewmats"]); Ks = _f32(scene["Ks"])
    return means, quats, scales, opac, colors, viewmats, Ks


def project(scene, opts: Options):
    """F1-F15 for every (camera, Gaussian).  Returns dense [C, N, ...] arrays."""
    means, quats, scales, opac, colors, viewmats, Ks = _scene_arrays(scene)
    N, C = means.shape[0], viewmats.shape[0]
    W, H = int(scene["width"]), int(scene["height"])
    K = colors.shape[1] if colors.ndim == 3 else 1
    out = dict(
        radii=np.zeros((C, N, 2), np.int32), mean2d_f=np.zeros((C, N, 2), np.float32),
        depth_f=np.zeros((C, N), np.float32), dec=np.zeros((C, N, 4), np.float32),
        mean2d=np.zeros((C, N, 2)), depth=np.zeros((C, N)),
        conic=np.zeros((C, N, 3)), comp=np.zeros((C, N)), opac_eff=np.zeros((C, N)),
        rgb=np.zeros((C, N, 3)))
    o = opts.c()
    lib().or_project(ct.byref(o), N, C, W, H, _p(means), _p(quats), _p(scales), _p(opac), _p(colors), K,
                     _p(viewmats), _p(Ks), _p(out["radii"]), _p(out["mean2d_f"]), _p(out["depth_f"]),
                     _p(out["dec"]), _p(out["mean2d"]), _p(out["depth"]), _p(out["conic"]), _p(out["comp"]),
                     _p(out["opac_eff"]), _p(out["rgb"]))
    return out


def isect(proj, C, N, W, H, opts: Options):
    """I1-I4 by brute-force enumeration + sort.  Returns keys (u64), ids (i32), offsets."""
    o = opts.c()
    radii, m2, d = proj["radii"], proj["mean2d_f"], proj["depth_f"]
    M = lib().or_isect(ct.byref(o), C, N, W, H, _p(radii), _p(m2), _p(d), 0, None, None, None)
    TS = opts.tile_size
    TX, TY = (W + TS - 1) // TS, (H + TS - 1) // TS
    keys = np.zeros(max(M, 1), np.uint64)
    ids = np.zeros(max(M, 1), np.int32)
    offs = np.zeros(C * TX * TY + 1, np.int32)
    M2 = lib().or_isect(ct.byref(o), C, N, W, H, _p(radii), _p(m2), _p(d), M, _p(keys), _p(ids), _p(offs))
    assert M2 == M
    return keys[:M], ids[:M], offs


def _depth64(proj):
    """fp64 depth t_z of every (c,n) (hand-built projections may give only the fp32 one)."""
    return _f64(proj["depth"] if "depth" in proj else proj["depth_f"])


def _flips(flips):
    return None if flips is None else np.ascontiguousarray(flips, np.uint32)


def render_fwd(proj, C, N, W, H, opts: Options, backgrounds=None, tile_mask=None, flips=None):
    """R1-R3 per pixel.  Also returns the accumulated depth sum z alpha T ("depth")
    and the expected depth ("depth_exp" = that sum / sum alpha T, with
    sum alpha T = 1 - T_final; 0 where nothing composited).  "ambig" [C,H,W] counts the
    ambiguous decisions (DESIGN Q28b) met per pixel; flips [C,H,W] (uint32, optional) takes
    the alternative outcome of the j-th of them where bit j is set (resolve_ambiguous)."""
    o = opts.c()
    bg = None if backgrounds is None else _f64(backgrounds)
    tm = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    out = dict(rgb=np.zeros((C, H, W, 3)), alpha=np.zeros((C, H, W)), T=np.zeros((C, H, W)),
               last_gid=np.zeros((C, H, W), np.int64), ambig=np.zeros((C, H, W), np.uint8),
               ncontrib=np.zeros((C, H, W), np.int32), depth=np.zeros((C, H, W)))
    lib().or_render_fwd(ct.byref(o), C, N, W, H, _p(proj["radii"]), _p(proj["mean2d_f"]), _p(proj["depth_f"]),
                        _p(proj["dec"]), _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["opac_eff"]), _p(proj["rgb"]), _p(bg),
                        _p(tm), _p(out["rgb"]), _p(out["alpha"]), _p(out["T"]), _p(out["last_gid"]),
                        _p(out["ambig"]), _p(out["ncontrib"]), _p(_depth64(proj)), _p(out["depth"]),
                        _p(_flips(flips)))
    A = 1.0 - out["T"]
    out["depth_exp"] = np.where(A > 0, out["depth"] / np.where(A > 0, A, 1.0), 0.0)
    return out


def render_pixels(proj, C, N, W, H, opts: Options, cams, pxs, pys, flips, backgrounds=None, feats=None):
    """R1-R3 for single pixels (cams[q], pxs[q], pys[q]) under the decision outcomes flips[q]
    (see render_fwd).  Returns colour [Q, 3 or D], T [Q], last_gid [Q] and namb [Q], the number
    of ambiguous decisions that walk met -- the enumeration of the outcomes an ambiguous pixel
    admits (DESIGN Q28b).  feats [N, D]: N-D feature mode (render_fwd_nd)."""
    rows, o = proj["rgb"], opts
    D = 3
    if feats is not None:
        feats = _f64(feats)
        D = feats.shape[1]
        rows = np.ascontiguousarray(np.broadcast_to(feats[None], (C, N, D)).reshape(C * N, D))
        o = _nd_opts(opts, D)
    Q = len(cams)
    out = dict(rgb=np.zeros((Q, D)), T=np.zeros(Q), last_gid=np.zeros(Q, np.int64), namb=np.zeros(Q, np.int32))
    bg = None if backgrounds is None else _f64(backgrounds)
    oc = o.c()
    lib().or_render_pixels(ct.byref(oc), C, N, W, H, _p(proj["radii"]), _p(proj["mean2d_f"]), _p(proj["depth_f"]),
                           _p(proj["dec"]), _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["opac_eff"]), _p(_f64(rows)),
                           _p(bg), Q, _p(np.ascontiguousarray(cams, np.int32)),
                           _p(np.ascontiguousarray(pxs, np.int32)), _p(np.ascontiguousarray(pys, np.int32)),
                           _p(np.ascontiguousarray(flips, np.uint32)), _p(out["rgb"]), _p(out["T"]),
                           _p(out["last_gid"]), _p(out["namb"]))
    return out


def render_bwd(proj, C, N, W, H, opts: Options, v_img, v_alpha=None, backgrounds=None, tile_mask=None,
               v_depth=None, v_depth_exp=None, flips=None):
    """B1-B6.  Returns v2d [C,N,9] (v_mean2d 2, v_conic 3, v_rgb 3, v_opac_eff 1), and for the
    parity tolerance (not part of the result): a2d, the sum over pixels of |per-pixel term|
    with B4's v_alpha replaced by the magnitudes of its parts (fp32 cancellation floor),
    s2d, the first-order change of each gradient for a 1-ulp shift of the fp32 projected
    means the kernel works with, g_ambig and the T-replay error.
    Depth rendering: v_depth = dL/d(accumulated depth) [C,H,W] and/or
    v_depth_exp = dL/d(expected depth); the expected depth D/A (A = 1 - T_final = sum alpha T)
    enters by the quotient rule, dL/dD += v_exp / A and dL/dA += -v_exp D / A^2 (the alpha
    output's gradient, Q26).  vz [C,N] = dL/d(depth of each (c,n)) (+ az, sz floors).
    absgrad [C,N,2] = sum over pixels of |dL_pixel/dmu'| per axis (App. Absgrad)."""
    o = opts.c()
    bg = None if backgrounds is None else _f64(backgrounds)
    tm = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    v_img = _f64(v_img)
    va = None if v_alpha is None else _f64(v_alpha)
    vD = None if v_depth is None else _f64(v_depth).copy()
    if v_depth_exp is not None:
        f = render_fwd(proj, C, N, W, H, opts, backgrounds, tile_mask, flips=flips)
        A = 1.0 - f["T"]
        ok = A > 0
        Ar = np.where(ok, A, 1.0)
        ve = _f64(v_depth_exp)
        vD = (np.zeros((C, H, W)) if vD is None else vD) + np.where(ok, ve / Ar, 0.0)
        va = (np.zeros((C, H, W)) if va is None else va.copy()) + np.where(ok, -ve * f["depth"] / (Ar * Ar), 0.0)
    v2d = np.zeros((C, N, 9)); a2d = np.zeros((C, N, 9)); s2d = np.zeros((C, N, 9)); absg = np.zeros((C, N, 2))
    vz = np.zeros((C, N)); az = np.zeros((C, N)); sz = np.zeros((C, N))
    amb = np.zeros((C, N), np.uint8)
    n2d = np.zeros((C, N), np.int32)
    d2d = np.zeros((C, N, 9))
    err = ct.c_double(0)
    lib().or_render_bwd(ct.byref(o), C, N, W, H, _p(proj["radii"]), _p(proj["mean2d_f"]), _p(proj["depth_f"]),
                        _p(proj["dec"]), _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["opac_eff"]), _p(proj["rgb"]), _p(bg),
                        _p(tm), _p(v_img), _p(va), _p(v2d), _p(a2d), _p(s2d), _p(amb), ct.byref(err),
                        _p(_depth64(proj)), _p(vD), _p(vz), _p(az), _p(sz), None, _p(absg), None, _p(_flips(flips)),
                        _p(n2d), _p(d2d), None)
    return dict(v2d=v2d, a2d=a2d, s2d=s2d, g_ambig=amb, T_replay_err=err.value, vz=vz, az=az, sz=sz, absgrad=absg,
                n2d=n2d, d2d=d2d)


def _nd_opts(opts: Options, D: int) -> Options:
    from dataclasses import replace
    return replace(opts, channels=int(D))


def render_fwd_nd(proj, feats, C, N, W, H, opts: Options, backgrounds=None, tile_mask=None, flips=None):
    """N-dimensional rasterization: the same R1-R3 composite with the per-Gaussian
    D-channel features feats [N, D] (camera independent) in place of the projected RGB.
    Returns feats image "feat" [C,H,W,D] plus alpha, T, last_gid, ambig as render_fwd."""
    feats = _f64(feats)
    D = feats.shape[1]
    rows = np.ascontiguousarray(np.broadcast_to(feats[None], (C, N, D)).reshape(C * N, D))
    p2 = dict(proj)
    p2["rgb"] = rows
    o = _nd_opts(opts, D).c()
    bg = None if backgrounds is None else _f64(backgrounds)
    tm = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    out = dict(feat=np.zeros((C, H, W, D)), alpha=np.zeros((C, H, W)), T=np.zeros((C, H, W)),
               last_gid=np.zeros((C, H, W), np.int64), ambig=np.zeros((C, H, W), np.uint8),
               ncontrib=np.zeros((C, H, W), np.int32))
    lib().or_render_fwd(ct.byref(o), C, N, W, H, _p(proj["radii"]), _p(proj["mean2d_f"]), _p(proj["depth_f"]),
                        _p(proj["dec"]), _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["opac_eff"]), _p(rows), _p(bg),
                        _p(tm), _p(out["feat"]), _p(out["alpha"]), _p(out["T"]), _p(out["last_gid"]),
                        _p(out["ambig"]), _p(out["ncontrib"]), None, None, _p(_flips(flips)))
    return out


def render_bwd_nd(proj, feats, C, N, W, H, opts: Options, v_feat, v_alpha=None, backgrounds=None, tile_mask=None,
                  flips=None):
    """B1-B6 with D-channel features: v2d (mean2d, conic, opac_eff slots; the rgb slots 0),
    vfeat [C,N,D] = dL/d(features of each (c,n)), and the tolerance models a2d, s2d and
    afeat (the sum over pixels of |per-pixel feature term|; a_colors its sum over cameras).
    The per-Gaussian feature gradient is vfeat summed over cameras (features are
    camera independent)."""
    feats = _f64(feats)
    D = feats.shape[1]
    rows = np.ascontiguousarray(np.broadcast_to(feats[None], (C, N, D)).reshape(C * N, D))
    o = _nd_opts(opts, D).c()
    bg = None if backgrounds is None else _f64(backgrounds)
    tm = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    va = None if v_alpha is None else _f64(v_alpha)
    v2d = np.zeros((C, N, 9)); a2d = np.zeros((C, N, 9)); s2d = np.zeros((C, N, 9)); absg = np.zeros((C, N, 2))
    vfeat = np.zeros((C, N, D)); afeat = np.zeros((C, N, D)); sfeat = np.zeros((C, N, D))
    amb = np.zeros((C, N), np.uint8)
    n2d = np.zeros((C, N), np.int32)
    d2d = np.zeros((C, N, 9))
    err = ct.c_double(0)
    lib().or_render_bwd(ct.byref(o), C, N, W, H, _p(proj["radii"]), _p(proj["mean2d_f"]), _p(proj["depth_f"]),
                        _p(proj["dec"]), _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["opac_eff"]), _p(rows), _p(bg),
                        _p(tm), _p(_f64(v_feat)), _p(va), _p(v2d), _p(a2d), _p(s2d), _p(amb), ct.byref(err),
                        None, None, None, None, None, _p(vfeat), _p(absg), _p(afeat), _p(_flips(flips)), _p(n2d),
                        _p(d2d), _p(sfeat))
    return dict(v2d=v2d, a2d=a2d, s2d=s2d, g_ambig=amb, T_replay_err=err.value, vfeat=vfeat, absgrad=absg, n2d=n2d, d2d=d2d,
                v_colors=vfeat.sum(axis=0), afeat=afeat, a_colors=afeat.sum(axis=0), s_colors=sfeat.sum(axis=0))


def project_bwd(scene, proj, v2d, opts: Options, vz=None, pose=False):
    """P1-P9, summed over cameras.  Returns v_means, v_quats, v_scales, v_opacities, v_colors
    (f64); vz [C,N] = dL/d depth (depth rendering) enters through t_z; pose=True also
    returns v_viewmats [C,4,4] (App. pose optimisation: the t, the
    Sigma_c = W Sigma W^T and the SH view-direction campos = -W^T w paths)."""
    means, quats, scales, opac, colors, viewmats, Ks = _scene_arrays(scene)
    N, C = means.shape[0], viewmats.shape[0]
    W, H = int(scene["width"]), int(scene["height"])
    K = colors.shape[1] if colors.ndim == 3 else 1
    o = opts.c()
    out = dict(v_means=np.zeros((N, 3)), v_quats=np.zeros((N, 4)), v_scales=np.zeros((N, 3)),
               v_opacities=np.zeros(N), v_colors=np.zeros(colors.shape))
    if pose:
        out["v_viewmats"] = np.zeros((C, 4, 4))
    lib().or_project_bwd(ct.byref(o), N, C, W, H, _p(means), _p(quats), _p(scales), _p(opac), _p(colors), K,
                         _p(viewmats), _p(Ks), _p(proj["radii"]), _p(_f64(v2d)), _p(out["v_means"]),
                         _p(out["v_quats"]), _p(out["v_scales"]), _p(out["v_opacities"]), _p(out["v_colors"]),
                         _p(None if vz is None else _f64(vz)), _p(out.get("v_viewmats")), 0)
    return out


def project_bwd_bound(scene, proj, e2d, opts: Options, ez=None, pose=False):
    """Tolerance model (not a result): the projection backward P1-P9 with every operand
    replaced by its magnitude and every subtraction by an addition, applied to the
    non-negative per-(c,n) bounds e2d [C,N,9] (and ez [C,N] for the depth slot).  Because
    P1-P9 are linear in (v2d, vz), this is |Jacobian| e, an upper bound on the change of each
    parameter gradient when every 2D gradient element moves by at most e; with e = |v2d| it
    is the sum of the magnitudes of the terms of each output (its fp32 rounding floor)."""
    means, quats, scales, opac, colors, viewmats, Ks = _scene_arrays(scene)
    N, C = means.shape[0], viewmats.shape[0]
    W, H = int(scene["width"]), int(scene["height"])
    K = colors.shape[1] if colors.ndim == 3 else 1
    o = opts.c()
    out = dict(v_means=np.zeros((N, 3)), v_quats=np.zeros((N, 4)), v_scales=np.zeros((N, 3)),
               v_opacities=np.zeros(N), v_colors=np.zeros(colors.shape))
    if pose:
        out["v_viewmats"] = np.zeros((C, 4, 4))
    e2d = np.abs(_f64(e2d))
    lib().or_project_bwd(ct.byref(o), N, C, W, H, _p(means), _p(quats), _p(scales), _p(opac), _p(colors), K,
                         _p(viewmats), _p(Ks), _p(proj["radii"]), _p(e2d), _p(out["v_means"]),
                         _p(out["v_quats"]), _p(out["v_scales"]), _p(out["v_opacities"]), _p(out["v_colors"]),
                         _p(None if ez is None else np.abs(_f64(ez))), _p(out.get("v_viewmats")), 1)
    return out


def project_bwd_clamp_alt(scene, proj, v2d, opts: Options, pose=False):
    """Tolerance model (not a result): the bound (project_bwd_bound) of the colour path of
    every SH channel whose clamp colour = max(0, raw) (Q22) is decided within the fp32
    rounding of raw -- both outcomes are correct there, and this is the magnitude of the
    difference between them in each parameter gradient."""
    means, quats, scales, opac, colors, viewmats, Ks = _scene_arrays(scene)
    N, C = means.shape[0], viewmats.shape[0]
    W, H = int(scene["width"]), int(scene["height"])
    K = colors.shape[1] if colors.ndim == 3 else 1
    o = opts.c()
    out = dict(v_means=np.zeros((N, 3)), v_quats=np.zeros((N, 4)), v_scales=np.zeros((N, 3)),
               v_opacities=np.zeros(N), v_colors=np.zeros(colors.shape))
    if pose:
        out["v_viewmats"] = np.zeros((C, 4, 4))
    lib().or_project_bwd(ct.byref(o), N, C, W, H, _p(means), _p(quats), _p(scales), _p(opac), _p(colors), K,
                         _p(viewmats), _p(Ks), _p(proj["radii"]), _p(np.abs(_f64(v2d))), _p(out["v_means"]),
                         _p(out["v_quats"]), _p(out["v_scales"]), _p(out["v_opacities"]), _p(out["v_colors"]),
                         None, _p(out.get("v_viewmats")), 2)
    return out


def pack(proj):
    """Packed mode (BASELINE configs[4]): the visible (c,n) pairs of the
    dense [C,N] layout in camera-major, then Gaussian order -- the definition written out
    (row-major nonzero of the visibility mask).  Returns (camera_ids, gaussian_ids) and the
    dense->packed index map (-1 where culled)."""
    r = proj["radii"]
    vis = (r[..., 0] > 0) & (r[..., 1] > 0)
    cam, gid = np.nonzero(vis)              # C order: camera-major, then n
    index = np.full(vis.shape, -1, np.int64)
    index[cam, gid] = np.arange(cam.size)
    return cam.astype(np.int32), gid.astype(np.int32), index


def forward_backward(scene, opts: Options, v_img, v_alpha=None, backgrounds=None, tile_mask=None,
                     with_isect=True):
    """The whole path: project -> isect -> render fwd -> render bwd -> project bwd."""
    C, N = scene["viewmats"].shape[0], scene["means"].shape[0]
    W, H = int(scene["width"]), int(scene["height"])
    proj = project(scene, opts)
    res = dict(proj=proj)
    if with_isect:
        res["keys"], res["ids"], res["offsets"] = isect(proj, C, N, W, H, opts)
    res["fwd"] = render_fwd(proj, C, N, W, H, opts, backgrounds, tile_mask)
    res["bwd"] = render_bwd(proj, C, N, W, H, opts, v_img, v_alpha, backgrounds, tile_mask)
    res["grads"] = project_bwd(scene, proj, res["bwd"]["v2d"], opts)
    return res


def densify_stats(radii, v_mean2d, scale=(1.0, 1.0), radius_scale=1.0):
    """Densification statistics (App. ADC P:196-200 and Absgrad P:204-206):
    per Gaussian n, over the cameras c where it is visible (radii > 0),
        grad2d[n] = sum_c || (sx g_x, sy g_y) ||,  g = that view's dL/dmu' (or its Absgrad sums)
        count[n]  = number of such cameras,  max_radii[n] = max_c max(rx, ry) * radius_scale.
    radii [C,N,2], v_mean2d [C,N,2].  The definition written out (Q37)."""
    radii = np.asarray(radii)
    vis = (radii[..., 0] > 0) & (radii[..., 1] > 0)
    g = _f64(v_mean2d) * np.asarray(scale, np.float64)
    norms = np.sqrt((g * g).sum(axis=-1))
    grad2d = np.where(vis, norms, 0.0).sum(axis=0)
    count = vis.sum(axis=0).astype(np.int64)
    max_radii = np.where(vis, radii.max(axis=-1), 0).max(axis=0) * float(radius_scale)
    return dict(grad2d=grad2d, count=count, max_radii=max_radii.astype(np.float64))
