"""Helpers shared by the GPU parity tests: run the CUDA path through the C-ABI (Engine)
and the oracle on the same seeded inputs, and compare with the tolerances of DESIGN.md
"Parity contract".  Nothing here computes any of the method's arithmetic."""
from __future__ import annotations

import numpy as np

# ---- tolerances ----
IMG_ATOL = 1e-4          # north_star: images and transmittance within 1e-4 absolute
GRAD_RTOL = 1e-3         # north_star: gradients within 1e-3 relative ...
GRAD2D_FLOOR = 1e-5      # ... plus this fraction of sum |per-pixel term| (fp32 atomics: 1e-5 A)


def to_torch(scene, device):
    import torch
    keys = ["means", "quats", "scales", "opacities", "colors", "viewmats", "Ks"]
    return tuple(torch.from_numpy(np.ascontiguousarray(scene[k], dtype=np.float32)).to(device) for k in keys)


def run_gpu(scene, *, antialiased=False, v_img=None, v_alpha=None, backgrounds=None, absgrad=False, device="cuda",
            cap=None, packed=False, nnz_capacity=None, depth_mode=0, v_depth=None, pose=False, **opt):
    import torch
    from paper_2409_06765_b200 import Engine
    C, N = scene["viewmats"].shape[0], scene["means"].shape[0]
    W, H = int(scene["width"]), int(scene["height"])
    deg = int(scene["sh_degree"])
    K = scene["colors"].shape[1] if deg >= 0 else None
    eng = Engine(N, C, W, H, sh_degree=deg, K=K, antialiased=antialiased, device=device, absgrad=absgrad,
                 with_keys=True, M_capacity=cap, packed=packed, nnz_capacity=nnz_capacity, depth_mode=depth_mode,
                 pose=pose, **opt)
    params = to_torch(scene, device)
    if v_img is None:
        v_img = np.zeros((C, H, W, 3), np.float32)
    v = torch.from_numpy(np.ascontiguousarray(v_img, dtype=np.float32)).to(device)
    va = None if v_alpha is None else torch.from_numpy(np.ascontiguousarray(v_alpha, np.float32)).to(device)
    bg = None if backgrounds is None else torch.from_numpy(np.ascontiguousarray(backgrounds, np.float32)).to(device)
    vd = None if v_depth is None else torch.from_numpy(np.ascontiguousarray(v_depth, np.float32)).to(device)
    eng.run_checked(params, v, va, bg, vd)
    torch.cuda.synchronize()
    M = eng.n_isect
    out = dict(
        M=M, radii=eng.radii.cpu().numpy(), splats=eng.splats.cpu().numpy(),
        ids=eng.isect_ids[:M].cpu().numpy(), keys=eng.isect_keys[:M].cpu().numpy().view(np.uint64),
        offsets=eng.tile_offsets.cpu().numpy(), rgb=eng.out_rgb.cpu().numpy(), alpha=eng.out_alpha.cpu().numpy(),
        T=eng.out_T.cpu().numpy(), last_ids=eng.last_ids.cpu().numpy(), v_splats=eng.v_splats.cpu().numpy(),
        v_means=eng.v_means.cpu().numpy(), v_quats=eng.v_quats.cpu().numpy(), v_scales=eng.v_scales.cpu().numpy(),
        v_opacities=eng.v_opacities.cpu().numpy(), v_colors=eng.v_colors.cpu().numpy(), engine=eng)
    if depth_mode:
        out["depth"] = eng.out_depth.cpu().numpy()
    if pose:
        out["v_viewmats"] = eng.v_viewmats.cpu().numpy()
    if packed:
        nnz = int(eng.nnz.item())
        out.update(nnz=nnz, camera_ids=eng.camera_ids[:nnz].cpu().numpy(),
                   gaussian_ids=eng.gaussian_ids[:nnz].cpu().numpy())
        for k in ("radii", "splats", "v_splats"):
            out[k] = out[k][:nnz]
    return out


def unpack(packed_rows, cam, gid, C, N):
    """Scatter packed per-item rows back into the dense [C, N, ...] layout (zeros elsewhere)."""
    dense = np.zeros((C, N) + packed_rows.shape[1:], packed_rows.dtype)
    dense[cam, gid] = packed_rows
    return dense


def last_gid(gpu, N):
    """Flat id of the last composited splat per pixel (-1 if none) from the GPU's last_ids."""
    C, H, W = gpu["last_ids"].shape
    TX = (W + 15) // 16
    TY = (H + 15) // 16
    ys, xs = np.mgrid[0:H, 0:W]
    tile = (ys // 16) * TX + (xs // 16)
    out = np.full((C, H, W), -1, np.int64)
    for c in range(C):
        start = gpu["offsets"][c * TX * TY + tile]
        li = gpu["last_ids"][c]
        has = li >= start
        rec = gpu["ids"][li[has]]
        if "camera_ids" in gpu:   # packed: record index -> flat id c*N + n
            rec = gpu["camera_ids"][rec].astype(np.int64) * N + gpu["gaussian_ids"][rec]
        out[c][has] = rec
    return out


def v2d_from_splats(v_splats):
    """GPU v_splats gradient slots (include/gs.h: mean2d 0-1, opac 2, conic 3-5, rgb 6-8) -> the
    oracle's 9-value layout (mean2d 2, conic 3, rgb 3, opac 1)."""
    vs = v_splats
    return np.concatenate([vs[..., 0:2], vs[..., 3:6], vs[..., 6:9], vs[..., 2:3]], axis=-1)


GRAD2D_ULP = 2.0          # ... plus this multiple of the 1-ulp(mu') sensitivity s2d


def check_grad2d(g, r, a, comparable, s=None, d=None):
    """|g - r| <= GRAD_RTOL |r| + GRAD2D_FLOOR * a + GRAD2D_ULP * s + d on comparable (c,n);
    d = the oracle's d2d, the difference between the outcomes of ambiguous alpha_max
    decisions (both correct, DESIGN Q28b)."""
    m = comparable[..., None] & np.ones_like(r, bool)
    tol = GRAD_RTOL * np.abs(r) + GRAD2D_FLOOR * a + 1e-12
    if s is not None:
        tol = tol + GRAD2D_ULP * s
    if d is not None:
        tol = tol + d
    bad = (np.abs(g - r) > tol) & m
    return bad


# ---- ambiguous pixels (DESIGN Q28b): every decision outcome within the fp32 error bound is
# a correct result; the GPU's pixel must equal one of the outcomes the oracle enumerates -----
MAX_OUTCOMES = 64         # outcomes tried per ambiguous pixel
MAX_ALT_PIXELS = 256      # pixels whose image-equal outcomes are bounded one by one


def resolve_ambiguous(proj, C, N, W, H, o, f, img, T, last, backgrounds=None, feats=None, atol=IMG_ATOL):
    """For every pixel where the oracle met an ambiguous decision (f["ambig"] > 0), enumerate
    the decision outcomes (flip masks, oracle.render_fwd) and pick the one closest to the
    GPU's pixel (colour and T; the last composited splat must be the GPU's), which must be
    within atol.  Every candidate value is computed by the oracle; the GPU's output only
    selects among them (a membership test).  Returns (flips [C,H,W] uint32, unresolved
    [C,H,W] bool, stats)."""
    import oracle
    key = "feat" if feats is not None else "rgb"
    amb = f["ambig"] > 0
    flips = np.zeros((C, H, W), np.uint32)
    unresolved = np.zeros((C, H, W), bool)
    todo = np.argwhere(amb)
    stats = dict(pixels=int(amb.size), ambiguous=int(amb.sum()), default=0, flipped=0, unresolved=0,
                 alternatives={})
    if len(todo) == 0:
        return flips, unresolved, stats
    cams, ys, xs = todo[:, 0], todo[:, 1], todo[:, 2]
    g_img, g_T, g_last = img[cams, ys, xs], T[cams, ys, xs], last[cams, ys, xs]

    def err(c_img, c_T, c_last, i):
        e = np.maximum(np.abs(c_img - g_img[i]).max(axis=-1), np.abs(c_T - g_T[i]))
        return np.where(c_last == g_last[i], e, np.inf)

    idx = np.arange(len(todo))
    best = err(f[key][cams, ys, xs], f["T"][cams, ys, xs], f["last_gid"][cams, ys, xs], idx)
    best_m = np.zeros(len(todo), np.int64)
    matching = [[0] if best[i] <= atol else [] for i in range(len(todo))]   # every outcome within atol
    namb0 = f["ambig"][cams, ys, xs].astype(np.int64)
    # candidates: every non-empty subset of the first k ambiguous decisions, extended when a
    # flipped walk meets further ambiguous decisions
    cand = [list(range(1, 1 << min(int(k), 6))) for k in namb0]
    tried = [set([0]) for _ in todo]
    for _ in range(4):
        q_pix, q_mask = [], []
        for i, ms in enumerate(cand):
            for m in ms:
                if m not in tried[i] and len(tried[i]) < MAX_OUTCOMES:
                    tried[i].add(m)
                    q_pix.append(i)
                    q_mask.append(m)
        if not q_pix:
            break
        q_pix = np.array(q_pix)
        r = oracle.render_pixels(proj, C, N, W, H, o, cams[q_pix], xs[q_pix], ys[q_pix], np.array(q_mask, np.uint32),
                                 backgrounds=backgrounds, feats=feats)
        e = err(r[key if key == "rgb" else "rgb"], r["T"], r["last_gid"], q_pix)
        cand = [[] for _ in todo]
        for j, (i, m) in enumerate(zip(q_pix, q_mask)):
            if e[j] <= atol:
                matching[i].append(m)
            if e[j] < best[i]:
                best[i], best_m[i] = e[j], m
            for b in range(max(int(namb0[i]), int(m).bit_length()), min(int(r["namb"][j]), 32)):
                cand[i].append(m | (1 << b))
    ok = best <= atol
    flips[cams, ys, xs] = np.where(ok, best_m, 0).astype(np.uint32)
    unresolved[cams[~ok], ys[~ok], xs[~ok]] = True
    stats["default"] = int((ok & (best_m == 0)).sum())
    stats["flipped"] = int((ok & (best_m != 0)).sum())
    stats["unresolved"] = int((~ok).sum())
    # pixels whose image does not tell two admitted outcomes apart: the gradient of either is
    # correct (oracle_reference widens the tolerance by their difference)
    stats["alternatives"] = {tuple(int(x) for x in todo[i]): [m for m in matching[i] if m != best_m[i]]
                             for i in range(len(todo)) if ok[i] and len(matching[i]) > 1}
    return flips, unresolved, stats


def oracle_reference(sc, o, gpu, v_img, v_alpha=None, backgrounds=None, tile_mask=None, with_isect=True,
                     proj=None, depth_mode=0, v_depth=None, pose=False, feats=None, img=None):
    """The oracle's whole path on the GPU run's inputs, with every ambiguous pixel resolved to
    the decision outcome the GPU took (resolve_ambiguous): forward, backward of the full loss
    (no pixel masked) and projection backward.  Depth rendering (depth_mode 1 accumulated /
    2 expected, v_depth its upstream gradient), pose gradients, N-D features (feats [N, D],
    img = the GPU's feature image) as in the oracle's API.  ref["amb"] carries the
    statistics; the caller asserts ref["unresolved"] is empty."""
    import oracle
    C, N = sc["viewmats"].shape[0], sc["means"].shape[0]
    W, H = int(sc["width"]), int(sc["height"])
    p = oracle.project(sc, o) if proj is None else proj
    bg = None if backgrounds is None else np.asarray(backgrounds, np.float64)
    va = None if v_alpha is None else np.asarray(v_alpha, np.float64)
    lg = last_gid(gpu, N)
    if feats is not None:
        f0 = oracle.render_fwd_nd(p, feats, C, N, W, H, o, bg, tile_mask)
        flips, unres, stats = resolve_ambiguous(p, C, N, W, H, o, f0, img, gpu["T"], lg, backgrounds=bg, feats=feats)
        f = oracle.render_fwd_nd(p, feats, C, N, W, H, o, bg, tile_mask, flips=flips) if flips.any() else f0
        b = oracle.render_bwd_nd(p, feats, C, N, W, H, o, np.asarray(v_img, np.float64), va, bg, tile_mask,
                                 flips=flips)
    else:
        f0 = oracle.render_fwd(p, C, N, W, H, o, bg, tile_mask)
        flips, unres, stats = resolve_ambiguous(p, C, N, W, H, o, f0, gpu["rgb"] if img is None else img, gpu["T"],
                                                lg, backgrounds=bg)
        f = oracle.render_fwd(p, C, N, W, H, o, bg, tile_mask, flips=flips) if flips.any() else f0
        kw = {}
        if depth_mode == 1:
            kw["v_depth"] = np.asarray(v_depth, np.float64)
        elif depth_mode == 2:
            kw["v_depth_exp"] = np.asarray(v_depth, np.float64)
        b = oracle.render_bwd(p, C, N, W, H, o, np.asarray(v_img, np.float64), va, bg, tile_mask, flips=flips, **kw)
    if tile_mask is not None:
        stats["pixels"] = int(np.repeat(np.repeat(np.asarray(tile_mask, bool), 16, 1), 16, 2)[:, :H, :W].sum())
    # outcomes the image cannot tell apart: widen each gradient tolerance by the difference of
    # the pixel's backward in the two outcomes (the loss restricted to that pixel, its tile only)
    alts = stats.pop("alternatives")
    stats["image_equal_outcomes"] = len(alts)
    b["dz"] = np.zeros_like(b["vz"]) if "vz" in b else None
    if feats is not None:
        b["d_colors"] = np.zeros_like(b["v_colors"])
    TX = (W + 15) // 16
    for (c, y, x), masks in list(alts.items())[:MAX_ALT_PIXELS]:
        vq = np.zeros_like(np.asarray(v_img, np.float64))
        vq[c, y, x] = v_img[c, y, x]
        vaq = None
        if va is not None:
            vaq = np.zeros_like(va)
            vaq[c, y, x] = va[c, y, x]
        tm = np.zeros((C, (H + 15) // 16, TX), np.uint8)
        tm[c, y // 16, x // 16] = 1
        outs = []
        for m in [int(flips[c, y, x])] + masks:
            fl = flips.copy()
            fl[c, y, x] = m
            if feats is not None:
                outs.append(oracle.render_bwd_nd(p, feats, C, N, W, H, o, vq, vaq, bg, tm, flips=fl))
            else:
                kw = {}
                if depth_mode:
                    vdq = np.zeros((C, H, W))
                    vdq[c, y, x] = v_depth[c, y, x]
                    kw["v_depth" if depth_mode == 1 else "v_depth_exp"] = vdq
                outs.append(oracle.render_bwd(p, C, N, W, H, o, vq, vaq, bg, tm, flips=fl, **kw))
        for alt in outs[1:]:
            b["d2d"] += np.abs(alt["v2d"] - outs[0]["v2d"])
            if b["dz"] is not None:
                b["dz"] += np.abs(alt["vz"] - outs[0]["vz"])
            if feats is not None:
                b["d_colors"] += np.abs(alt["v_colors"] - outs[0]["v_colors"])
    if len(alts) > MAX_ALT_PIXELS:
        unres = unres.copy()
        for (c, y, x) in list(alts)[MAX_ALT_PIXELS:]:
            unres[c, y, x] = True   # too many to bound: reported as unresolved
    ref = dict(proj=p, fwd=f, bwd=b, flips=flips, unresolved=unres, amb=stats, opts=o)
    ref["grads"] = oracle.project_bwd(sc, p, b["v2d"], o, vz=b["vz"] if depth_mode else None, pose=pose)
    if with_isect:
        ref["keys"], ref["ids"], ref["offsets"] = oracle.isect(p, C, N, W, H, o)
    return ref


def report(label, ref, **extra):
    """Appends the parity statistics of one comparison to $GS_PARITY_REPORT (JSON lines)."""
    import json
    import os
    path = os.environ.get("GS_PARITY_REPORT")
    if not path:
        return
    with open(path, "a") as fh:
        fh.write(json.dumps(dict(test=label, amb=ref["amb"], **extra)) + "\n")


GRAD_KEYS = ("v_means", "v_quats", "v_scales", "v_opacities", "v_colors")


def assert_grads(sc, gpu, ref, label="", packed=False, pose=False, depth=False, keys=GRAD_KEYS, vs=None):
    """The gradient contract against a resolved oracle reference (oracle_reference): every
    2D record-gradient element of every visible (c,n) within GRAD_RTOL |r| + the oracle's
    floors (check_grad2d), the depth slot likewise, every parameter-gradient element within
    GRAD_RTOL |r| + its propagated floor (grad3d_tolerance), pose per entry."""
    p, b, o = ref["proj"], ref["bwd"], ref["opts"]
    C, N = sc["viewmats"].shape[0], sc["means"].shape[0]
    if vs is None:
        vs = gpu["v_splats"]
        if packed:
            vs = unpack(vs, gpu["camera_ids"], gpu["gaussian_ids"], C, N)
    vis = p["radii"][..., 0] > 0
    g2 = v2d_from_splats(vs)
    bad = check_grad2d(g2, b["v2d"], b["a2d"], vis, b["s2d"], b["d2d"])
    if bad.any():
        rows = [dict(idx=[int(x) for x in ix], g=float(g2[tuple(ix)]), r=float(b["v2d"][tuple(ix)]),
                     a=float(b["a2d"][tuple(ix)]), s=float(b["s2d"][tuple(ix)]), d=float(b["d2d"][tuple(ix)]),
                     n2d=int(b["n2d"][tuple(ix[:2])]), g_ambig=int(b["g_ambig"][tuple(ix[:2])]))
                for ix in np.argwhere(bad)[:6]]
        raise AssertionError(f"{label}: 2D grads: {int(bad.sum())} bad of {int(vis.sum()) * 9}: {rows}")
    if depth:
        badz = check_grad2d(vs[..., 9:10], b["vz"][..., None], b["az"][..., None], vis, b["sz"][..., None],
                            b["dz"][..., None])
        assert not badz.any(), f"{label}: depth grads: {int(badz.sum())} bad"
    floors = grad3d_tolerance(sc, p, o, b, pose=pose, depth=depth)
    worst = {}
    for k in keys:
        nbad, w, rel = check_grad3d_elementwise(gpu[k], ref["grads"][k], floors[k])
        assert nbad == 0, f"{label}: {k}: {nbad} elements out of tolerance (worst {w:.3f} of it)"
        assert rel <= GRAD_RTOL, (label, k, rel)
        worst[k] = round(w, 4)
    if pose:
        g, r, fl = gpu["v_viewmats"][:, :3], ref["grads"]["v_viewmats"][:, :3], floors["v_viewmats"][:, :3]
        nbad, w, _ = check_grad3d_elementwise(g, r, fl)
        assert nbad == 0, f"{label}: pose: {nbad} entries out of tolerance (worst {w:.3f})"
        assert np.all(gpu["v_viewmats"][:, 3] == 0)
        worst["v_viewmats"] = round(w, 4)
    report(label, ref, worst_tolerance_used=worst)
    return worst


def assert_images(gpu, ref, sel=None, label="", img=None, key="rgb", atol=IMG_ATOL):
    """Every (selected) pixel: colour, T and alpha within atol of the resolved oracle image,
    the last composited splat identical; no ambiguous pixel left unresolved."""
    assert not ref["unresolved"].any(), f"{label}: " + amb_report(ref)
    f = ref["fwd"]
    N = ref["proj"]["radii"].shape[1]
    if sel is None:
        sel = np.ones(f["T"].shape, bool)
    im = gpu["rgb"] if img is None else img
    assert np.abs(im - f[key])[sel].max() <= atol, label
    assert np.abs(gpu["T"] - f["T"])[sel].max() <= IMG_ATOL, label
    if "alpha" in gpu:
        assert np.abs(gpu["alpha"] - f["alpha"])[sel].max() <= IMG_ATOL, label
    assert np.array_equal(last_gid(gpu, N)[sel], f["last_gid"][sel]), label


def amb_report(ref):
    s = ref["amb"]
    return (f"ambiguous pixels {s['ambiguous']}/{s['pixels']} ({100.0 * s['ambiguous'] / max(s['pixels'], 1):.4f} %): "
            f"{s['default']} took the fp64 outcome, {s['flipped']} another admitted outcome, "
            f"{s['unresolved']} unresolved")


# ---- 3D (parameter) gradients: element-wise model --------------------------------------
# Per element |g - r| <= GRAD_RTOL |r| + B(GRAD2D_FLOOR a2d + GRAD2D_ULP s2d + d2d)
#                          + EPS3D B(|v2d|) + Bc,
# with B = oracle.project_bwd_bound (|Jacobian| of the projection backward): the 2D floors
# (and the ambiguous alpha_max outcomes) carried through the chain, the fp32 rounding of the
# chain itself relative to the sum of the magnitudes of its terms, and Bc the outcomes of
# ambiguous SH clamp decisions (oracle.project_bwd_clamp_alt).
EPS3D = 1e-5


def grad3d_tolerance(sc, p, o, b, pose=False, depth=False):
    """Per-element tolerance of every parameter-gradient tensor (dict), from the oracle's
    tolerance models (render_bwd's a2d / s2d and project_bwd_bound)."""
    import oracle
    e = GRAD2D_FLOOR * b["a2d"] + GRAD2D_ULP * b["s2d"] + b["d2d"]
    ez = GRAD2D_FLOOR * b["az"] + GRAD2D_ULP * b["sz"] + b["dz"] if depth else None
    Bf = oracle.project_bwd_bound(sc, p, e, o, ez=ez, pose=pose)
    Ba = oracle.project_bwd_bound(sc, p, np.abs(b["v2d"]), o, ez=np.abs(b["vz"]) if depth else None, pose=pose)
    Bc = oracle.project_bwd_clamp_alt(sc, p, b["v2d"], o, pose=pose)
    return {k: Bf[k] + EPS3D * Ba[k] + Bc[k] for k in Bf}


def check_grad3d_elementwise(g, r, floor):
    """Every element: |g - r| <= GRAD_RTOL |r| + floor.  Returns (n bad, worst ratio, rel L2)."""
    g = np.asarray(g, np.float64)
    err = np.abs(g - r)
    tol = GRAD_RTOL * np.abs(r) + floor + 1e-30
    rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
    return int((err > tol).sum()), float((err / tol).max()) if err.size else 0.0, rel


# ---- two GPU runs of the same kernels that differ only in the order of their fp32 atomic
# sums (sharded vs one GPU, opacity-aware vs 3-sigma bins, support test on vs off) --------
U32 = 2.0 ** -24


def atomic_order_tol2d(b):
    """|s_1 - s_2| <= 2 gamma_{n-1} sum |t_i| for two fp32 summation orders of the same n terms
    (gamma_k = k u / (1 - k u)); n = the oracle's term count n2d of each (c,n), sum |t_i| <=
    its a2d (magnitudes of B4's parts), + 8 u a2d for the fp32 evaluation of the terms."""
    n = np.maximum(b["n2d"].astype(np.float64) - 1, 0)[..., None]
    gam = n * U32 / (1 - n * U32)
    return (2 * gam + 8 * U32) * b["a2d"]


def assert_same_kernel_grads(sc, o, b, one, other, keys=GRAD_KEYS, label="", vs_one=None, vs_other=None,
                             depth=False, pose=False):
    """2D record gradients within the atomic-order bound; parameter gradients within that
    bound carried through the projection backward (K8 is deterministic in its inputs) plus
    its own fp32 rounding (2 EPS3D B(|v2d|)); the depth slot and pose likewise."""
    import oracle
    p = oracle.project(sc, o)
    vis = p["radii"][..., 0] > 0
    tol2 = atomic_order_tol2d(b)
    n = np.maximum(b["n2d"].astype(np.float64) - 1, 0)
    tolz = (2 * n * U32 / (1 - n * U32) + 8 * U32) * b["az"] if depth else None
    if vs_one is not None:
        g1, g2 = v2d_from_splats(vs_one), v2d_from_splats(vs_other)
        bad = (np.abs(g1 - g2) > tol2 + 1e-30) & vis[..., None]
        assert not bad.any(), f"{label}: 2D: {int(bad.sum())} elements beyond the atomic-order bound"
    Bt = oracle.project_bwd_bound(sc, p, tol2, o, ez=tolz, pose=pose)
    Ba = oracle.project_bwd_bound(sc, p, np.abs(b["v2d"]), o, ez=np.abs(b["vz"]) if depth else None, pose=pose)
    worst = {}
    for k in list(keys) + (["v_viewmats"] if pose else []):
        a1, a2 = np.asarray(one[k], np.float64), np.asarray(other[k], np.float64)
        bt, ba = Bt[k], Ba[k]
        if k == "v_viewmats":
            a1, a2, bt, ba = a1[:, :3], a2[:, :3], bt[:, :3], ba[:, :3]
        d = np.abs(a1 - a2)
        tol = bt + 2 * EPS3D * ba + 1e-30
        nb = int((d > tol).sum())
        assert nb == 0, f"{label}: {k}: {nb} elements beyond the atomic-order bound (worst {(d / tol).max():.3f})"
        worst[k] = round(float((d / tol).max()), 4)
    return worst
