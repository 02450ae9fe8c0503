"""The paper's user-level call (Fig. 1) on top of the C-ABI.

    render_colors, render_alphas, meta = rasterization(
        means, quats, scales, opacities, colors, viewmats, Ks, width, height)

Differentiable with respect to means, quats, scales, opacities and colors through a
torch.autograd.Function whose forward/backward call the library's kernels.  PyTorch
only allocates memory and provides the stream.  There is no CPU or PyTorch fallback:
inputs must be contiguous float32 CUDA tensors.
"""
from __future__ import annotations

import math

import torch

from . import _lib as L

# last intersection count per problem shape: the next call's capacity estimate
_M_CACHE: dict = {}


def _sh_degree_of(colors, sh_degree):
    if sh_degree is None:
        if colors.dim() == 2:
            return -1
        return int(round(math.sqrt(colors.shape[1]))) - 1
    return int(sh_degree)


class _Rasterize(torch.autograd.Function):
    @staticmethod
    def forward(ctx, means, quats, scales, opacities, colors, viewmats, Ks, backgrounds, cfg, absgrad_out):
        o = cfg["opts"]
        W, H = cfg["width"], cfg["height"]
        N, C = means.shape[0], viewmats.shape[0]
        K = cfg["K"]
        dev = means.device
        radii = torch.empty((C, N, 2), dtype=torch.int32, device=dev)
        splats = torch.empty((C, N, L.SPLAT_FLOATS), dtype=torch.float32, device=dev)
        L.gs_project(o, means, quats, scales, opacities, colors, K, viewmats, Ks, W, H, radii, splats)
        TX, TY = L.tiles(W, H)
        offs = torch.empty(C * TX * TY + 1, dtype=torch.int32, device=dev)
        Mdev = torch.zeros(1, dtype=torch.int64, device=dev)
        ovf = torch.zeros(1, dtype=torch.int32, device=dev)
        key = (N, C, W, H)
        cap = _M_CACHE.get(key, max(1024, 4 * C * N))
        while True:
            ids = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            wsz = L.gs_isect_workspace_size(C, N, W, H, cap)
            ws_raw = torch.empty(wsz + 256, dtype=torch.uint8, device=dev)
            a = (-ws_raw.data_ptr()) % 256
            L.gs_isect_tiles(o, C, N, W, H, radii, splats, cap, Mdev, ovf, ids, None, offs, ws_raw[a:a + wsz])
            M = int(Mdev.item())                      # one D->H read per call (as gsplat's .item())
            _M_CACHE[key] = math.ceil(M * 1.25) + 1024
            if int(ovf.item()) == 0:
                break
            cap = M + 1024
        out_rgb = torch.empty((C, H, W, 3), dtype=torch.float32, device=dev)
        out_alpha = torch.empty((C, H, W), dtype=torch.float32, device=dev)
        out_T = torch.empty((C, H, W), dtype=torch.float32, device=dev)
        last_ids = torch.empty((C, H, W), dtype=torch.int32, device=dev)
        L.gs_rasterize_fwd(o, C, N, W, H, splats, backgrounds, ids, offs, out_rgb, out_alpha, out_T, last_ids)
        ctx.save_for_backward(means, quats, scales, opacities, colors, viewmats, Ks, backgrounds, radii, splats,
                              ids, offs, out_T, last_ids)
        ctx.cfg = cfg
        ctx.absgrad_out = absgrad_out
        ctx.mark_non_differentiable(radii, splats, ids, offs, out_T, last_ids)
        return out_rgb, out_alpha, radii, splats, ids, offs, out_T, last_ids, Mdev

    @staticmethod
    def backward(ctx, v_rgb, v_alpha, *unused):
        (means, quats, scales, opacities, colors, viewmats, Ks, backgrounds, radii, splats, ids, offs, out_T,
         last_ids) = ctx.saved_tensors
        cfg = ctx.cfg
        o = cfg["opts"]
        W, H, K = cfg["width"], cfg["height"], cfg["K"]
        N, C = means.shape[0], viewmats.shape[0]
        v_rgb = v_rgb.contiguous() if v_rgb is not None else torch.zeros((C, H, W, 3), device=means.device)
        v_alpha = v_alpha.contiguous() if v_alpha is not None else None
        v_splats = torch.empty_like(splats)
        absgrad = ctx.absgrad_out is not None
        L.gs_rasterize_bwd(o, C, N, W, H, splats, backgrounds, ids, offs, out_T, last_ids, v_rgb, v_alpha, absgrad,
                           v_splats)
        if absgrad:
            ctx.absgrad_out.copy_(torch.stack([v_splats[..., 7], v_splats[..., 11]], dim=-1))
        v_means = torch.empty_like(means)
        v_quats = torch.empty_like(quats)
        v_scales = torch.empty_like(scales)
        v_opac = torch.empty_like(opacities)
        v_colors = torch.empty_like(colors)
        L.gs_project_bwd(o, means, quats, scales, opacities, colors, K, viewmats, Ks, W, H, radii, v_splats, v_means,
                         v_quats, v_scales, v_opac, v_colors)
        cfg["v_splats"] = v_splats
        return v_means, v_quats, v_scales, v_opac, v_colors, None, None, None, None, None


def rasterization(means, quats, scales, opacities, colors, viewmats, Ks, width, height, *, sh_degree=None,
                  near_plane=0.01, far_plane=1e10, eps2d=0.3, rasterize_mode="classic", tile_size=16,
                  backgrounds=None, alpha_max=0.99, absgrad=False, fov_clamp=True, bbox_mode=0):
    """Render C views of N Gaussians.

    means [N,3], quats [N,4] (w,x,y,z), scales [N,3] (activated), opacities [N] (activated),
    colors [N,3] (RGB, sh_degree None/-1) or [N,K,3] (SH), viewmats [C,4,4] (world->camera),
    Ks [C,3,3], backgrounds [C,3] or None.  rasterize_mode "classic" | "antialiased" (A.4).
    Returns render_colors [C,H,W,3], render_alphas [C,H,W,1] and a meta dict.
    """
    if rasterize_mode not in ("classic", "antialiased"):
        raise ValueError("rasterize_mode must be 'classic' or 'antialiased'")
    deg = _sh_degree_of(colors, sh_degree)
    K = colors.shape[1] if deg >= 0 else 1
    o = L.options(sh_degree=deg, antialiased=rasterize_mode == "antialiased", near_plane=near_plane,
                  far_plane=far_plane, eps2d=eps2d, alpha_max=alpha_max, tile_size=tile_size, bbox_mode=bbox_mode,
                  fov_clamp=fov_clamp)
    cfg = dict(opts=o, width=int(width), height=int(height), K=K)
    C, N = viewmats.shape[0], means.shape[0]
    absgrad_out = torch.zeros((C, N, 2), device=means.device) if absgrad else None
    args = [t.contiguous() if t is not None else None for t in (means, quats, scales, opacities, colors, viewmats, Ks,
                                                              backgrounds)]
    out_rgb, out_alpha, radii, splats, ids, offs, out_T, last_ids, Mdev = _Rasterize.apply(*args, cfg, absgrad_out)
    meta = dict(radii=radii, means2d=splats[..., 0:2], depths=splats[..., 3], conics=splats[..., 4:7],
                opacities=splats[..., 2], colors=splats[..., 8:11], splats=splats,
                isect_ids=ids, flatten_ids=ids, tile_offsets=offs, n_isects=Mdev, T_final=out_T, last_ids=last_ids,
                width=int(width), height=int(height), tile_size=tile_size, n_cameras=C, absgrad=absgrad_out,
                cfg=cfg)
    return out_rgb, out_alpha.unsqueeze(-1), meta
