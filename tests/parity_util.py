"""Helpers shared by the GPU parity tests: run the CUDA path through the C-ABI (Engine)
and the oracle on the same seeded inputs, and compare with the tolerances of DESIGN.md
"Parity contract".  Nothing here computes any of the method's arithmetic."""
from __future__ import annotations

import numpy as np

# ---- tolerances ----
IMG_ATOL = 1e-4          # north_star: images and transmittance within 1e-4 absolute
GRAD_RTOL = 1e-3         # north_star: gradients within 1e-3 relative ...
GRAD2D_FLOOR = 3e-5      # ... plus this fraction of sum |per-pixel term| (fp32 atomics)
GRAD3D_FLOOR = 1e-4      # ... or of max |g| of the tensor for the projection-chain outputs
MIN_COMPARABLE = 0.999   # fraction of visible Gaussians that must be comparable (not ambiguous)


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
        out[c][has] = gpu["ids"][li[has]]
    return out


def v2d_from_splats(v_splats):
    """GPU v_splats gradient slots (include/gs.h: mean2d 0-1, opac 2, conic 3-5, rgb 6-8) -> the
    oracle's 9-value layout (mean2d 2, conic 3, rgb 3, opac 1)."""
    vs = v_splats
    return np.concatenate([vs[..., 0:2], vs[..., 3:6], vs[..., 6:9], vs[..., 2:3]], axis=-1)


GRAD2D_ULP = 2.0          # ... plus this multiple of the 1-ulp(mu') sensitivity s2d


def check_grad2d(g, r, a, comparable, s=None):
    """|g - r| <= GRAD_RTOL |r| + GRAD2D_FLOOR * a + GRAD2D_ULP * s on comparable (c,n)."""
    m = comparable[..., None] & np.ones_like(r, bool)
    tol = GRAD_RTOL * np.abs(r) + GRAD2D_FLOOR * a + 1e-12
    if s is not None:
        tol = tol + GRAD2D_ULP * s
    bad = (np.abs(g - r) > tol) & m
    return bad


def check_grad3d(g, r, comparable_n):
    """Elementwise |g - r| <= GRAD_RTOL |r| + GRAD3D_FLOOR max|r| on comparable Gaussians;
    returns (bad mask, relative L2 error over comparable Gaussians)."""
    g = g.reshape(g.shape[0], -1).astype(np.float64)
    r = r.reshape(r.shape[0], -1)
    scale = np.abs(r[comparable_n]).max() if comparable_n.any() else 0.0
    bad = (np.abs(g - r) > GRAD_RTOL * np.abs(r) + GRAD3D_FLOOR * scale + 1e-30) & comparable_n[:, None]
    d = (g - r)[comparable_n]
    rr = r[comparable_n]
    rel = np.linalg.norm(d) / max(np.linalg.norm(rr), 1e-30)
    return bad, rel
