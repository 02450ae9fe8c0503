"""ctypes binding of libgsplat_b200 (include/gs.h) -- argument marshalling only.

Every step of the path runs in the library's CUDA kernels; this module converts torch
tensors to device pointers and the current CUDA stream to a cudaStream_t.  It fails
loudly when the shared library is missing or a tensor is not a contiguous CUDA tensor of
the expected dtype: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as ct
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgsplat_b200.so")
SPLAT_FLOATS = 12
ABI_VERSION = 11
# largest item / record count of one call: ids and capacities are int32 (include/gs.h)
MAX_ITEMS = (1 << 31) - 2048

GS_STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported", 3: "capacity exceeded", 4: "cuda error"}


class GsOptions(ct.Structure):
    _fields_ = [
        ("near_plane", ct.c_float), ("far_plane", ct.c_float), ("eps2d", ct.c_float),
        ("alpha_max", ct.c_float), ("alpha_min", ct.c_float), ("t_min", ct.c_float),
        ("tile_size", ct.c_int32), ("antialiased", ct.c_int32), ("sh_degree", ct.c_int32),
        ("bbox_mode", ct.c_int32), ("fov_clamp", ct.c_int32), ("packed", ct.c_int32),
        ("support_cull", ct.c_int32), ("bwd_zero_fill", ct.c_int32),
    ]


class GsError(RuntimeError):
    pass


_lib = None

# name -> (restype, argtypes)
_P, _I32, _I64, _SZ = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_size_t
SIGNATURES = {
    "gs_default_options": (None, [_P]),
    "gs_status_string": (ct.c_char_p, [_I32]),
    "gs_last_error": (ct.c_char_p, []),
    "gs_abi_version": (_I32, []),
    "gs_project": (_I32, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P]),
    "gs_isect_workspace_size": (_SZ, [_I32, _I64, _I32, _I32, _I64]),
    "gs_isect_tiles": (_I32, [_P, _I32, _I64, _I32, _I32, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "gs_rasterize_fwd": (_I32, [_P, _I32, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P]),
    "gs_rasterize_stats": (_I32, [_P, _I32, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "gs_rasterize_bwd": (_I32, [_P, _I32, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P,
                                _P, _P, _P]),
    "gs_tile_order": (_I32, [_P, _I32, _I32, _I32, _P, _P, _P]),
    "gs_zero_splat_grads": (_I32, [_P, _I32, _I64, _P, _P]),
    "gs_project_bwd_workspace_size": (_SZ, [_I64, _I32]),
    "gs_project_bwd": (_I32, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P,
                              _P, _P, _P, _P, _SZ, _P]),
    "gs_project_bwd_range": (_I32, [_P, _I64, _I64, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P,
                                    _P, _P, _P, _P, _P, _P]),
    "gs_rasterize_fwd_nd": (_I32, [_P, _I32, _I64, _I32, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "gs_rasterize_bwd_nd": (_I32, [_P, _I32, _I64, _I32, _I32, _P, _P, _I32, _P, _I64, _P, _P, _P, _P, _P, _P, _P,
                                   _I32, _P, _P, _P, _P]),
    "gs_project_packed_workspace_size": (_SZ, [_I64, _I32]),
    "gs_project_packed": (_I32, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _P, _P, _P,
                                 _P, _P, _P, _SZ, _P]),
    "gs_isect_packed_workspace_size": (_SZ, [_I32, _I64, _I32, _I32, _I64]),
    "gs_isect_tiles_packed": (_I32, [_P, _I32, _I64, _P, _I32, _I32, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _SZ,
                                     _P]),
    "gs_project_bwd_packed_workspace_size": (_SZ, [_I64, _I32]),
    "gs_project_bwd_packed": (_I32, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _P, _P,
                                     _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "gs_shard_pack": (_I32, [_I64, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "gs_shard_unpack": (_I32, [_I64, _P, _P, _P, _P, _P, _P]),
    "gs_densify_stats": (_I32, [_P, _I64, _I32, _I64, _P, _P, _P, _P, _I32, ct.c_float, ct.c_float, ct.c_float,
                                _P, _P, _P, _P]),
}


def lib():
    """Load libgsplat_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GsError(f"{LIB_PATH} is missing: build it with `python -m paper_2409_06765_b200.build` "
                          "(there is no CPU fallback)")
        L = ct.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.gs_abi_version() != ABI_VERSION:
            raise GsError("libgsplat_b200 ABI mismatch")
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().gs_last_error().decode()
        raise GsError(f"{what}: {GS_STATUS.get(status, status)} {msg}")


def options(sh_degree=3, antialiased=False, near_plane=0.01, far_plane=1e10, eps2d=0.3, alpha_max=0.99,
            alpha_min=1.0 / 255.0, t_min=1e-4, tile_size=16, bbox_mode=0, fov_clamp=True,
            packed=False, support_cull=True, bwd_zero_fill=True) -> GsOptions:
    o = GsOptions()
    lib().gs_default_options(ct.byref(o))
    o.near_plane, o.far_plane, o.eps2d = near_plane, far_plane, eps2d
    o.alpha_max, o.alpha_min, o.t_min = alpha_max, alpha_min, t_min
    o.tile_size, o.antialiased, o.sh_degree = tile_size, int(bool(antialiased)), int(sh_degree)
    o.bbox_mode, o.fov_clamp = int(bbox_mode), int(bool(fov_clamp))
    o.packed = int(bool(packed))
    o.support_cull = int(bool(support_cull))
    o.bwd_zero_fill = int(bool(bwd_zero_fill))
    return o


def ptr(t, dtype=torch.float32, name="tensor"):
    """Device pointer of a contiguous CUDA tensor of `dtype` (None -> NULL)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise GsError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise GsError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise GsError(f"{name} must be contiguous")
    return t.data_ptr()


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def tiles(width, height, tile=16):
    return (width + tile - 1) // tile, (height + tile - 1) // tile


# ------------------------------------------------------------------------------------
# Thin wrappers with the C names.  All tensors are caller-allocated.
# ------------------------------------------------------------------------------------
def gs_project(o, means, quats, scales, opacities, colors, K, viewmats, Ks, width, height, radii, splats,
               stream=None):
    N, C = means.shape[0], viewmats.shape[0]
    check(lib().gs_project(ct.byref(o), N, C, width, height, ptr(means, name="means"), ptr(quats, name="quats"),
                           ptr(scales, name="scales"), ptr(opacities, name="opacities"), ptr(colors, name="colors"),
                           K, ptr(viewmats, name="viewmats"), ptr(Ks, name="Ks"),
                           ptr(radii, torch.int32, "radii"), ptr(splats, name="splats"), stream_ptr(stream)),
          "gs_project")


def gs_isect_workspace_size(C, N, width, height, cap):
    return int(lib().gs_isect_workspace_size(C, N, width, height, cap))


def gs_isect_tiles(o, C, N, width, height, radii, splats, cap, M, overflow, isect_ids, isect_keys, tile_offsets,
                   workspace, stream=None):
    check(lib().gs_isect_tiles(ct.byref(o), C, N, width, height, ptr(radii, torch.int32, "radii"),
                               ptr(splats, name="splats"), cap, ptr(M, torch.int64, "M"),
                               ptr(overflow, torch.int32, "overflow"), ptr(isect_ids, torch.int32, "isect_ids"),
                               ptr(isect_keys, torch.int64, "isect_keys"),
                               ptr(tile_offsets, torch.int32, "tile_offsets"), ptr(workspace, torch.uint8, "ws"),
                               workspace.numel(), stream_ptr(stream)),
          "gs_isect_tiles")


def gs_rasterize_fwd(o, C, N, width, height, splats, backgrounds, isect_ids, tile_offsets, out_rgb, out_alpha,
                     out_T, last_ids, out_depth=None, depth_mode=0, isect_masks=None, stream=None):
    check(lib().gs_rasterize_fwd(ct.byref(o), C, N, width, height, ptr(splats, name="splats"),
                                 ptr(backgrounds, name="backgrounds"), ptr(isect_ids, torch.int32, "isect_ids"),
                                 ptr(tile_offsets, torch.int32, "tile_offsets"), ptr(out_rgb, name="out_rgb"),
                                 ptr(out_alpha, name="out_alpha"), ptr(out_T, name="out_T"),
                                 ptr(last_ids, torch.int32, "last_ids"), ptr(out_depth, name="out_depth"),
                                 int(depth_mode), ptr(isect_masks, torch.int16, "isect_masks"), stream_ptr(stream)),
          "gs_rasterize_fwd")


def gs_rasterize_stats(o, C, N, width, height, splats, isect_ids, tile_offsets, n_eval, n_contrib, terminated=None,
                       stream=None):
    check(lib().gs_rasterize_stats(ct.byref(o), C, N, width, height, ptr(splats, name="splats"),
                                   ptr(isect_ids, torch.int32, "isect_ids"),
                                   ptr(tile_offsets, torch.int32, "tile_offsets"), ptr(n_eval, torch.int32, "n_eval"),
                                   ptr(n_contrib, torch.int32, "n_contrib"), ptr(terminated, torch.int32, "terminated"),
                                   stream_ptr(stream)),
          "gs_rasterize_stats")


def gs_rasterize_bwd(o, C, N, width, height, splats, backgrounds, isect_ids, tile_offsets, out_T, last_ids,
                     v_out_rgb, v_out_alpha, absgrad, v_splats, out_depth=None, v_out_depth=None, depth_mode=0,
                     isect_masks=None, stream=None, tile_order=None):
    check(lib().gs_rasterize_bwd(ct.byref(o), C, N, width, height, ptr(splats, name="splats"),
                                 ptr(backgrounds, name="backgrounds"), ptr(isect_ids, torch.int32, "isect_ids"),
                                 ptr(tile_offsets, torch.int32, "tile_offsets"), ptr(out_T, name="out_T"),
                                 ptr(last_ids, torch.int32, "last_ids"), ptr(v_out_rgb, name="v_out_rgb"),
                                 ptr(v_out_alpha, name="v_out_alpha"), ptr(out_depth, name="out_depth"),
                                 ptr(v_out_depth, name="v_out_depth"), int(depth_mode), int(bool(absgrad)),
                                 ptr(isect_masks, torch.int16, "isect_masks"),
                                 ptr(tile_order, torch.int32, "tile_order"), ptr(v_splats, name="v_splats"),
                                 stream_ptr(stream)),
          "gs_rasterize_bwd")


def gs_zero_splat_grads(o, C, N, v_splats, stream=None):
    check(lib().gs_zero_splat_grads(ct.byref(o), C, N, ptr(v_splats, name="v_splats"), stream_ptr(stream)),
          "gs_zero_splat_grads")


def gs_tile_order(o, C, width, height, tile_offsets, tile_order, stream=None):
    check(lib().gs_tile_order(ct.byref(o), C, width, height, ptr(tile_offsets, torch.int32, "tile_offsets"),
                              ptr(tile_order, torch.int32, "tile_order"), stream_ptr(stream)), "gs_tile_order")


def gs_project_bwd_workspace_size(N, C):
    return int(lib().gs_project_bwd_workspace_size(N, C))


def gs_project_bwd(o, means, quats, scales, opacities, colors, K, viewmats, Ks, width, height, radii, v_splats,
                   v_means, v_quats, v_scales, v_opacities, v_colors, v_viewmats=None, workspace=None, stream=None):
    N, C = means.shape[0], viewmats.shape[0]
    check(lib().gs_project_bwd(ct.byref(o), N, C, width, height, ptr(means, name="means"), ptr(quats, name="quats"),
                               ptr(scales, name="scales"), ptr(opacities, name="opacities"),
                               ptr(colors, name="colors"), K, ptr(viewmats, name="viewmats"), ptr(Ks, name="Ks"),
                               ptr(radii, torch.int32, "radii"), ptr(v_splats, name="v_splats"),
                               ptr(v_means, name="v_means"), ptr(v_quats, name="v_quats"),
                               ptr(v_scales, name="v_scales"), ptr(v_opacities, name="v_opacities"),
                               ptr(v_colors, name="v_colors"), ptr(v_viewmats, name="v_viewmats"),
                               ptr(workspace, torch.uint8, "ws"), 0 if workspace is None else workspace.numel(),
                               stream_ptr(stream)),
          "gs_project_bwd")


def gs_project_bwd_range(o, n_begin, n_end, means, quats, scales, opacities, colors, K, viewmats, Ks, width, height,
                         radii, v_splats, v_means, v_quats, v_scales, v_opacities, v_colors, stream=None):
    """gs_project_bwd for the Gaussians [n_begin, n_end): the v_* tensors are that range's own
    rows (e.g. one gradient bucket)."""
    N, C = means.shape[0], viewmats.shape[0]
    check(lib().gs_project_bwd_range(ct.byref(o), N, n_begin, n_end, C, width, height, ptr(means, name="means"),
                                     ptr(quats, name="quats"), ptr(scales, name="scales"),
                                     ptr(opacities, name="opacities"), ptr(colors, name="colors"), K,
                                     ptr(viewmats, name="viewmats"), ptr(Ks, name="Ks"),
                                     ptr(radii, torch.int32, "radii"), ptr(v_splats, name="v_splats"),
                                     ptr(v_means, name="v_means"), ptr(v_quats, name="v_quats"),
                                     ptr(v_scales, name="v_scales"), ptr(v_opacities, name="v_opacities"),
                                     ptr(v_colors, name="v_colors"), stream_ptr(stream)),
          "gs_project_bwd_range")


# ---- packed mode (Q29) ------------------------------------------------------------------
def gs_project_packed_workspace_size(N, C):
    return int(lib().gs_project_packed_workspace_size(N, C))


def gs_project_packed(o, means, quats, scales, opacities, colors, K, viewmats, Ks, width, height, cap, nnz,
                      overflow, camera_ids, gaussian_ids, radii, splats, workspace, stream=None):
    N, C = means.shape[0], viewmats.shape[0]
    check(lib().gs_project_packed(ct.byref(o), N, C, width, height, ptr(means, name="means"),
                                  ptr(quats, name="quats"), ptr(scales, name="scales"),
                                  ptr(opacities, name="opacities"), ptr(colors, name="colors"), K,
                                  ptr(viewmats, name="viewmats"), ptr(Ks, name="Ks"), cap,
                                  ptr(nnz, torch.int64, "nnz"), ptr(overflow, torch.int32, "overflow"),
                                  ptr(camera_ids, torch.int32, "camera_ids"),
                                  ptr(gaussian_ids, torch.int32, "gaussian_ids"), ptr(radii, torch.int32, "radii"),
                                  ptr(splats, name="splats"), ptr(workspace, torch.uint8, "ws"), workspace.numel(),
                                  stream_ptr(stream)),
          "gs_project_packed")


def gs_isect_packed_workspace_size(C, cap_nnz, width, height, cap):
    return int(lib().gs_isect_packed_workspace_size(C, cap_nnz, width, height, cap))


def gs_isect_tiles_packed(o, C, cap_nnz, nnz, width, height, camera_ids, radii, splats, cap, M, overflow, isect_ids,
                          isect_keys, tile_offsets, workspace, stream=None):
    check(lib().gs_isect_tiles_packed(ct.byref(o), C, cap_nnz, ptr(nnz, torch.int64, "nnz"), width, height,
                                      ptr(camera_ids, torch.int32, "camera_ids"), ptr(radii, torch.int32, "radii"),
                                      ptr(splats, name="splats"), cap, ptr(M, torch.int64, "M"),
                                      ptr(overflow, torch.int32, "overflow"),
                                      ptr(isect_ids, torch.int32, "isect_ids"),
                                      ptr(isect_keys, torch.int64, "isect_keys"),
                                      ptr(tile_offsets, torch.int32, "tile_offsets"),
                                      ptr(workspace, torch.uint8, "ws"), workspace.numel(), stream_ptr(stream)),
          "gs_isect_tiles_packed")


def gs_project_bwd_packed_workspace_size(N, C):
    return int(lib().gs_project_bwd_packed_workspace_size(N, C))


def gs_project_bwd_packed(o, means, quats, scales, opacities, colors, K, viewmats, Ks, width, height, cap_nnz, nnz,
                          camera_ids, gaussian_ids, radii, v_splats, v_means, v_quats, v_scales, v_opacities,
                          v_colors, workspace, v_viewmats=None, stream=None):
    N, C = means.shape[0], viewmats.shape[0]
    check(lib().gs_project_bwd_packed(ct.byref(o), N, C, width, height, ptr(means, name="means"),
                                      ptr(quats, name="quats"), ptr(scales, name="scales"),
                                      ptr(opacities, name="opacities"), ptr(colors, name="colors"), K,
                                      ptr(viewmats, name="viewmats"), ptr(Ks, name="Ks"), cap_nnz,
                                      ptr(nnz, torch.int64, "nnz"), ptr(camera_ids, torch.int32, "camera_ids"),
                                      ptr(gaussian_ids, torch.int32, "gaussian_ids"),
                                      ptr(radii, torch.int32, "radii"), ptr(v_splats, name="v_splats"),
                                      ptr(v_means, name="v_means"), ptr(v_quats, name="v_quats"),
                                      ptr(v_scales, name="v_scales"), ptr(v_opacities, name="v_opacities"),
                                      ptr(v_colors, name="v_colors"), ptr(v_viewmats, name="v_viewmats"),
                                      ptr(workspace, torch.uint8, "ws"), workspace.numel(), stream_ptr(stream)),
          "gs_project_bwd_packed")


# ---- N-D features -----------------------------------------------------------
def gs_rasterize_fwd_nd(o, C, N, width, height, splats, feats, gaussian_ids, backgrounds, isect_ids, tile_offsets,
                        out_feats, out_alpha, out_T, last_ids, isect_masks=None, stream=None):
    D = feats.shape[1]
    check(lib().gs_rasterize_fwd_nd(ct.byref(o), C, N, width, height, ptr(splats, name="splats"),
                                    ptr(feats, name="feats"), D, ptr(gaussian_ids, torch.int32, "gaussian_ids"),
                                    ptr(backgrounds, name="backgrounds"), ptr(isect_ids, torch.int32, "isect_ids"),
                                    ptr(tile_offsets, torch.int32, "tile_offsets"), ptr(out_feats, name="out_feats"),
                                    ptr(out_alpha, name="out_alpha"), ptr(out_T, name="out_T"),
                                    ptr(last_ids, torch.int32, "last_ids"),
                                    ptr(isect_masks, torch.int16, "isect_masks"), stream_ptr(stream)),
          "gs_rasterize_fwd_nd")


def gs_rasterize_bwd_nd(o, C, N, width, height, splats, feats, gaussian_ids, n_gauss, backgrounds, isect_ids,
                        tile_offsets, out_T, last_ids, v_out_feats, v_out_alpha, absgrad, isect_masks, v_splats,
                        v_feats, stream=None):
    D = feats.shape[1]
    check(lib().gs_rasterize_bwd_nd(ct.byref(o), C, N, width, height, ptr(splats, name="splats"),
                                    ptr(feats, name="feats"), D, ptr(gaussian_ids, torch.int32, "gaussian_ids"),
                                    n_gauss, ptr(backgrounds, name="backgrounds"),
                                    ptr(isect_ids, torch.int32, "isect_ids"),
                                    ptr(tile_offsets, torch.int32, "tile_offsets"), ptr(out_T, name="out_T"),
                                    ptr(last_ids, torch.int32, "last_ids"), ptr(v_out_feats, name="v_out_feats"),
                                    ptr(v_out_alpha, name="v_out_alpha"), int(bool(absgrad)),
                                    ptr(isect_masks, torch.int16, "isect_masks"), ptr(v_splats, name="v_splats"),
                                    ptr(v_feats, name="v_feats"), stream_ptr(stream)),
          "gs_rasterize_bwd_nd")


# ---- Gaussian-sharded scale-out (NEXT-4(i)) ---------------------------------------
SHARD_ROW_FLOATS = 16


def gs_shard_pack(cap_nnz, nnz, C, view_starts, camera_ids, radii, splats, send, send_counts, stream=None):
    R = len(view_starts) - 1
    vs = (ct.c_int32 * (R + 1))(*[int(v) for v in view_starts])
    check(lib().gs_shard_pack(cap_nnz, ptr(nnz, torch.int64, "nnz"), C, R, ct.cast(vs, ct.c_void_p),
                              ptr(camera_ids, torch.int32, "camera_ids"), ptr(radii, torch.int32, "radii"),
                              ptr(splats, name="splats"), ptr(send, name="send"),
                              ptr(send_counts, torch.int64, "send_counts"), stream_ptr(stream)),
          "gs_shard_pack")


def gs_shard_unpack(n_recv, recv, camera_ids, radii, splats, nnz, stream=None):
    check(lib().gs_shard_unpack(int(n_recv), ptr(recv, name="recv"), ptr(camera_ids, torch.int32, "camera_ids"),
                                ptr(radii, torch.int32, "radii"), ptr(splats, name="splats"),
                                ptr(nnz, torch.int64, "nnz"), stream_ptr(stream)),
          "gs_shard_unpack")


# ---- densification statistics (NEXT-1; App. ADC, Absgrad P:204-206) -------------
def gs_densify_stats(o, N, C, radii, v_splats, grad2d, count, max_radii, absgrad=False, scale=(1.0, 1.0),
                     radius_scale=1.0, nnz_capacity=0, nnz=None, gaussian_ids=None, stream=None):
    check(lib().gs_densify_stats(ct.byref(o), N, C, nnz_capacity, ptr(nnz, torch.int64, "nnz"),
                                 ptr(gaussian_ids, torch.int32, "gaussian_ids"), ptr(radii, torch.int32, "radii"),
                                 ptr(v_splats, name="v_splats"), int(bool(absgrad)), float(scale[0]),
                                 float(scale[1]), float(radius_scale), ptr(grad2d, name="grad2d"),
                                 ptr(count, torch.int32, "count"), ptr(max_radii, name="max_radii"),
                                 stream_ptr(stream)),
          "gs_densify_stats")
