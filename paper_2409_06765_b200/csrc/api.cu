// C-ABI entry points of libgsplat_b200 (include/gs.h): argument validation and dispatch to
// the stage launchers.  No allocation, no host synchronisation, no global mutable state
// except the per-thread last-error string.
#include <stdio.h>
#include <string.h>

#include "gs_internal.cuh"

namespace gsb {
static thread_local char g_err[512] = "";
void set_last_error(const char* where, cudaError_t e) {
    snprintf(g_err, sizeof g_err, "%s: %s", where, cudaGetErrorString(e));
}
}  // namespace gsb

namespace {

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }
inline bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

gs_status check_opts(const gs_options* o) {
    if (!o) return GS_ERR_INVALID_ARGUMENT;
    if (o->tile_size != GS_TILE) return GS_ERR_UNSUPPORTED;
    if (o->sh_degree < -1 || o->sh_degree > 3) return GS_ERR_INVALID_ARGUMENT;
    if (!(o->eps2d >= 0.f) || !(o->alpha_max > 0.f) || !(o->alpha_max < 1.f) || !(o->alpha_min >= 0.f) ||
        !(o->t_min >= 0.f) || !(o->near_plane > 0.f))
        return GS_ERR_INVALID_ARGUMENT;
    if (o->bbox_mode < 0 || o->bbox_mode > 2 || o->packed < 0 || o->packed > 1) return GS_ERR_INVALID_ARGUMENT;
    if (o->support_cull < 0 || o->support_cull > 1) return GS_ERR_INVALID_ARGUMENT;
    if (o->bwd_zero_fill < 0 || o->bwd_zero_fill > 1) return GS_ERR_INVALID_ARGUMENT;
    return GS_OK;
}

gs_status check_dims(int64_t N, int32_t C, int32_t W, int32_t H) {
    if (N < 0 || C < 1 || W < 1 || H < 1) return GS_ERR_INVALID_ARGUMENT;
    if ((int64_t)C * N >= (int64_t)1 << 31) return GS_ERR_INVALID_ARGUMENT;   // flat ids are int32
    const int64_t TT = (int64_t)((W + GS_TILE - 1) / GS_TILE) * ((H + GS_TILE - 1) / GS_TILE);
    if (TT * C >= (int64_t)1 << 31) return GS_ERR_INVALID_ARGUMENT;
    return GS_OK;
}

// Raster calls: in packed mode N is the total record count and record ids are packed indices
// < N, so only N itself (not C*N) must fit the int32 ids (Q29)
gs_status check_raster_dims(const gs_options* o, int64_t N, int32_t C, int32_t W, int32_t H) {
    if (o->packed) {
        gs_status s = check_dims(N, 1, W, H);
        return s != GS_OK ? s : check_dims(0, C, W, H);
    }
    return check_dims(N, C, W, H);
}

}  // namespace

#define GS_TRY(x)                     \
    do {                              \
        gs_status st_ = (x);          \
        if (st_ != GS_OK) return st_; \
    } while (0)
#define GS_REQ(cond)                                        \
    do {                                                    \
        if (!(cond)) return GS_ERR_INVALID_ARGUMENT;        \
    } while (0)

extern "C" {

void gs_default_options(gs_options* o) {
    if (!o) return;
    o->near_plane = 0.01f;
    o->far_plane = 1e10f;
    o->eps2d = 0.3f;
    o->alpha_max = 0.99f;
    o->alpha_min = 1.f / 255.f;
    o->t_min = 1e-4f;
    o->tile_size = GS_TILE;
    o->antialiased = 0;
    o->sh_degree = 3;
    o->bbox_mode = 0;
    o->fov_clamp = 1;
    o->packed = 0;
    o->support_cull = 1;
    o->bwd_zero_fill = 1;
}

const char* gs_status_string(int32_t s) {
    switch (s) {
        case GS_OK: return "ok";
        case GS_ERR_INVALID_ARGUMENT: return "invalid argument";
        case GS_ERR_UNSUPPORTED: return "unsupported";
        case GS_ERR_CAPACITY: return "capacity exceeded";
        case GS_ERR_CUDA: return "cuda error";
        default: return "unknown status";
    }
}

const char* gs_last_error(void) { return gsb::g_err; }
int32_t gs_abi_version(void) { return GS_ABI_VERSION; }

gs_status gs_project(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height, const float* means,
                     const float* quats, const float* scales, const float* opacities, const float* colors, int32_t K,
                     const float* viewmats, const float* Ks, int32_t* radii, float* splats, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 0);
    GS_TRY(check_dims(N, C, width, height));
    if (N == 0) return GS_OK;
    GS_REQ(means && quats && scales && opacities && viewmats && Ks && radii && splats);
    GS_REQ(colors || opt->sh_degree < 0);   // NULL direct colours: N-D feature mode
    GS_REQ(aligned16(quats) && aligned16(splats) && aligned8(radii) && aligned4(means) && aligned4(scales) &&
           aligned4(opacities) && aligned4(colors) && aligned4(viewmats) && aligned4(Ks));
    if (opt->sh_degree >= 0) GS_REQ(K >= (opt->sh_degree + 1) * (opt->sh_degree + 1));
    return gsb::launch_project_fwd(*opt, N, C, width, height, means, quats, scales, opacities, colors,
                                   opt->sh_degree >= 0 ? K : 1, viewmats, Ks, radii, splats,
                                   static_cast<cudaStream_t>(stream));
}

size_t gs_isect_workspace_size(int32_t C, int64_t N, int32_t width, int32_t height, int64_t M_capacity) {
    if (C < 1 || N < 0 || width < 1 || height < 1 || M_capacity < 0) return 0;
    return gsb::isect_workspace_bytes((int64_t)C * N, M_capacity);
}

gs_status gs_isect_tiles(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                         const int32_t* radii, const float* splats, int64_t M_capacity, int64_t* M, int32_t* overflow,
                         int32_t* isect_ids, uint64_t* isect_keys, int32_t* tile_offsets, void* workspace,
                         size_t workspace_bytes, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 0);
    GS_TRY(check_dims(N, C, width, height));
    GS_REQ(M_capacity >= 0 && M_capacity < ((int64_t)1 << 31) - 1);
    GS_REQ(M && overflow && tile_offsets && workspace);
    GS_REQ(N == 0 || (radii && splats));
    GS_REQ(M_capacity == 0 || isect_ids);
    GS_REQ(aligned8(M) && aligned4(overflow) && aligned4(tile_offsets) && aligned4(isect_ids) &&
           aligned8(isect_keys) && (reinterpret_cast<uintptr_t>(workspace) & 255u) == 0);
    GS_REQ(N == 0 || (aligned8(radii) && aligned16(splats)));
    GS_REQ(workspace_bytes >= gsb::isect_workspace_bytes((int64_t)C * N, M_capacity));
    return gsb::launch_isect(*opt, C, N, width, height, radii, splats, (int64_t)C * N, nullptr, nullptr, M_capacity, M,
                             overflow, isect_ids, isect_keys, tile_offsets, workspace, workspace_bytes,
                             static_cast<cudaStream_t>(stream));
}

gs_status gs_rasterize_fwd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                           const float* splats, const float* backgrounds, const int32_t* isect_ids,
                           const int32_t* tile_offsets, float* out_rgb, float* out_alpha, float* out_T,
                           int32_t* last_ids, float* out_depth, int32_t depth_mode, uint16_t* isect_masks,
                           void* stream) {
    GS_TRY(check_opts(opt));
    GS_TRY(check_raster_dims(opt, N, C, width, height));
    GS_REQ(tile_offsets && out_rgb && out_alpha && out_T && last_ids);
    GS_REQ(!out_depth || depth_mode == 1 || depth_mode == 2);
    GS_REQ(aligned16(splats) && aligned4(isect_ids) && aligned4(backgrounds) && aligned4(out_rgb) &&
           aligned4(out_alpha) && aligned4(out_T) && aligned4(last_ids) && aligned4(out_depth));
    return gsb::launch_raster_fwd(*opt, C, N, width, height, splats, backgrounds, isect_ids, tile_offsets, out_rgb,
                                  out_alpha, out_T, last_ids, out_depth, depth_mode, isect_masks,
                                  static_cast<cudaStream_t>(stream));
}

gs_status gs_rasterize_stats(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                             const float* splats, const int32_t* isect_ids, const int32_t* tile_offsets,
                             int32_t* n_eval, int32_t* n_contrib, int32_t* terminated, void* stream) {
    GS_TRY(check_opts(opt));
    GS_TRY(check_raster_dims(opt, N, C, width, height));
    GS_REQ(tile_offsets && n_eval && n_contrib);
    GS_REQ(aligned16(splats) && aligned4(isect_ids) && aligned4(n_eval) && aligned4(n_contrib) && aligned4(terminated));
    return gsb::launch_raster_stats(*opt, C, N, width, height, splats, isect_ids, tile_offsets, n_eval, n_contrib,
                                    terminated,
                                    static_cast<cudaStream_t>(stream));
}

gs_status gs_rasterize_bwd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                           const float* splats, const float* backgrounds, const int32_t* isect_ids,
                           const int32_t* tile_offsets, const float* out_T, const int32_t* last_ids,
                           const float* v_out_rgb, const float* v_out_alpha, const float* out_depth,
                           const float* v_out_depth, int32_t depth_mode, int32_t absgrad,
                           const uint16_t* isect_masks, const int32_t* tile_order, float* v_splats, void* stream) {
    GS_TRY(check_opts(opt));
    GS_TRY(check_raster_dims(opt, N, C, width, height));
    GS_REQ(tile_offsets && out_T && last_ids && v_out_rgb && (v_splats || N == 0));
    GS_REQ(!v_out_depth || depth_mode == 1 || (depth_mode == 2 && out_depth));
    GS_REQ(aligned16(splats) && aligned16(v_splats) && aligned4(isect_ids) && aligned4(backgrounds) &&
           aligned4(out_T) && aligned4(last_ids) && aligned4(v_out_rgb) && aligned4(v_out_alpha) &&
           aligned4(out_depth) && aligned4(v_out_depth) && aligned4(tile_order));
    return gsb::launch_raster_bwd(*opt, C, N, width, height, splats, backgrounds, isect_ids, tile_offsets, out_T,
                                  last_ids, v_out_rgb, v_out_alpha, out_depth, v_out_depth, depth_mode, absgrad,
                                  isect_masks, tile_order, v_splats, static_cast<cudaStream_t>(stream));
}

gs_status gs_zero_splat_grads(const gs_options* opt, int32_t C, int64_t N, float* v_splats, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(N >= 0 && C >= 1 && (v_splats || N == 0) && aligned16(v_splats));
    const size_t nrec = opt->packed ? (size_t)N : (size_t)C * (size_t)N;
    return gsb::launch_zero_splat_grads(v_splats, nrec, static_cast<cudaStream_t>(stream));
}

gs_status gs_tile_order(const gs_options* opt, int32_t C, int32_t width, int32_t height,
                        const int32_t* tile_offsets, int32_t* tile_order, void* stream) {
    GS_TRY(check_opts(opt));
    GS_TRY(check_dims(0, C, width, height));
    GS_REQ(tile_offsets && tile_order && aligned4(tile_offsets) && aligned4(tile_order));
    return gsb::launch_tile_order(C, width, height, tile_offsets, tile_order, static_cast<cudaStream_t>(stream));
}

size_t gs_project_bwd_workspace_size(int64_t N, int32_t C) {
    if (N < 0 || C < 1) return 0;
    return gsb::project_bwd_workspace_bytes(N, C);
}

gs_status gs_project_bwd(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                         const float* means, const float* quats, const float* scales, const float* opacities,
                         const float* colors, int32_t K, const float* viewmats, const float* Ks, const int32_t* radii,
                         const float* v_splats, float* v_means, float* v_quats, float* v_scales, float* v_opacities,
                         float* v_colors, float* v_viewmats, void* workspace, size_t workspace_bytes, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 0);
    GS_TRY(check_dims(N, C, width, height));
    GS_REQ(aligned4(v_viewmats));
    if (v_viewmats)
        GS_REQ(workspace && (reinterpret_cast<uintptr_t>(workspace) & 255u) == 0 &&
               workspace_bytes >= gsb::project_bwd_workspace_bytes(N, C));
    if (N > 0) {
        GS_REQ(means && quats && scales && opacities && viewmats && Ks && radii && v_splats && v_means &&
               v_quats && v_scales && v_opacities && (opt->sh_degree < 0 || (colors && v_colors)));
        GS_REQ(aligned16(quats) && aligned16(v_quats) && aligned16(v_splats) && aligned8(radii) && aligned4(means) &&
               aligned4(v_means) && aligned4(colors) && aligned4(v_colors) && aligned4(scales) && aligned4(v_scales));
        if (opt->sh_degree >= 0) GS_REQ(K >= (opt->sh_degree + 1) * (opt->sh_degree + 1));
    }
    return gsb::launch_project_bwd(*opt, N, C, width, height, means, quats, scales, opacities, colors,
                                   opt->sh_degree >= 0 ? K : 1, viewmats, Ks, radii, v_splats, v_means, v_quats,
                                   v_scales, v_opacities, v_colors, v_viewmats, workspace,
                                   static_cast<cudaStream_t>(stream));
}

gs_status gs_project_bwd_range(const gs_options* opt, int64_t N, int64_t n_begin, int64_t n_end, int32_t C,
                               int32_t width, int32_t height, const float* means, const float* quats,
                               const float* scales, const float* opacities, const float* colors, int32_t K,
                               const float* viewmats, const float* Ks, const int32_t* radii, const float* v_splats,
                               float* v_means, float* v_quats, float* v_scales, float* v_opacities, float* v_colors,
                               void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 0);
    GS_TRY(check_dims(N, C, width, height));
    GS_REQ(0 <= n_begin && n_begin <= n_end && n_end <= N);
    if (n_end > n_begin) {
        GS_REQ(means && quats && scales && opacities && viewmats && Ks && radii && v_splats && v_means &&
               v_quats && v_scales && v_opacities && (opt->sh_degree < 0 || (colors && v_colors)));
        GS_REQ(aligned16(quats) && aligned16(v_quats) && aligned16(v_splats) && aligned8(radii) && aligned4(means) &&
               aligned4(v_means) && aligned4(colors) && aligned4(v_colors) && aligned4(scales) && aligned4(v_scales));
        if (opt->sh_degree >= 0) GS_REQ(K >= (opt->sh_degree + 1) * (opt->sh_degree + 1));
    }
    return gsb::launch_project_bwd_range(*opt, N, n_begin, n_end, C, width, height, means, quats, scales, opacities,
                                         colors, opt->sh_degree >= 0 ? K : 1, viewmats, Ks, radii, v_splats, v_means,
                                         v_quats, v_scales, v_opacities, v_colors, static_cast<cudaStream_t>(stream));
}

// ---- N-D features ------------------------------------------------------

gs_status gs_rasterize_fwd_nd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                              const float* splats, const float* feats, int32_t D, const int32_t* gaussian_ids,
                              const float* backgrounds, const int32_t* isect_ids, const int32_t* tile_offsets,
                              float* out_feats, float* out_alpha, float* out_T, int32_t* last_ids,
                              uint16_t* isect_masks, void* stream) {
    GS_TRY(check_opts(opt));
    GS_TRY(check_raster_dims(opt, N, C, width, height));
    GS_REQ(D >= 1 && feats && tile_offsets && out_feats && out_alpha && out_T && last_ids);
    GS_REQ(!opt->packed || gaussian_ids);
    GS_REQ(aligned16(splats) && aligned4(feats) && aligned4(gaussian_ids) && aligned4(isect_ids) &&
           aligned4(backgrounds) && aligned4(out_feats) && aligned4(out_alpha) && aligned4(out_T) &&
           aligned4(last_ids));
    return gsb::launch_raster_fwd_nd(*opt, C, N, width, height, splats, feats, D,
                                     opt->packed ? gaussian_ids : nullptr, backgrounds, isect_ids, tile_offsets,
                                     out_feats, out_alpha, out_T, last_ids, isect_masks,
                                     static_cast<cudaStream_t>(stream));
}

gs_status gs_rasterize_bwd_nd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                              const float* splats, const float* feats, int32_t D, const int32_t* gaussian_ids,
                              int64_t n_gauss, const float* backgrounds, const int32_t* isect_ids,
                              const int32_t* tile_offsets, const float* out_T, const int32_t* last_ids,
                              const float* v_out_feats, const float* v_out_alpha, int32_t absgrad,
                              const uint16_t* isect_masks, float* v_splats, float* v_feats, void* stream) {
    GS_TRY(check_opts(opt));
    GS_TRY(check_raster_dims(opt, N, C, width, height));
    GS_REQ(D >= 1 && n_gauss >= 0 && feats && tile_offsets && out_T && last_ids && v_out_feats);
    if (absgrad && D > 4) return GS_ERR_UNSUPPORTED;   // |v_mean2d| per pixel needs every channel in one pass
    GS_REQ((v_splats || N == 0) && (v_feats || n_gauss == 0));
    GS_REQ(!opt->packed || gaussian_ids);
    GS_REQ(opt->packed || n_gauss == N);
    GS_REQ(aligned16(splats) && aligned16(v_splats) && aligned4(feats) && aligned4(gaussian_ids) &&
           aligned4(isect_ids) && aligned4(backgrounds) && aligned4(out_T) && aligned4(last_ids) &&
           aligned4(v_out_feats) && aligned4(v_out_alpha) && aligned4(v_feats));
    return gsb::launch_raster_bwd_nd(*opt, C, N, width, height, splats, feats, D,
                                     opt->packed ? gaussian_ids : nullptr, n_gauss, backgrounds, isect_ids,
                                     tile_offsets, out_T, last_ids, v_out_feats, v_out_alpha, absgrad, isect_masks,
                                     v_splats, v_feats, static_cast<cudaStream_t>(stream));
}

// ---- packed mode (Q29) ----------------------------------------------------------------

size_t gs_project_packed_workspace_size(int64_t N, int32_t C) {
    if (N < 0 || C < 1) return 0;
    return gsb::project_packed_workspace_bytes(N, C);
}

gs_status gs_project_packed(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                            const float* means, const float* quats, const float* scales, const float* opacities,
                            const float* colors, int32_t K, const float* viewmats, const float* Ks,
                            int64_t nnz_capacity, int64_t* nnz, int32_t* overflow, int32_t* camera_ids,
                            int32_t* gaussian_ids, int32_t* radii, float* splats, void* workspace,
                            size_t workspace_bytes, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 1);
    GS_TRY(check_raster_dims(opt, N, C, width, height));   // packed: item ids < 2^31, not C*N
    GS_REQ(nnz_capacity >= 0 && nnz_capacity < ((int64_t)1 << 31) - 1);
    GS_REQ(nnz && overflow && workspace && aligned8(nnz) && aligned4(overflow));
    GS_REQ((reinterpret_cast<uintptr_t>(workspace) & 255u) == 0);
    GS_REQ(workspace_bytes >= gsb::project_packed_workspace_bytes(N, C));
    GS_REQ(N == 0 || (means && quats && scales && opacities && viewmats && Ks && (colors || opt->sh_degree < 0)));
    GS_REQ(nnz_capacity == 0 || (camera_ids && gaussian_ids && radii && splats));
    GS_REQ(aligned16(quats) && aligned16(splats) && aligned8(radii) && aligned4(camera_ids) &&
           aligned4(gaussian_ids) && aligned4(means) && aligned4(scales) && aligned4(opacities) &&
           aligned4(colors) && aligned4(viewmats) && aligned4(Ks));
    if (opt->sh_degree >= 0) GS_REQ(K >= (opt->sh_degree + 1) * (opt->sh_degree + 1));
    return gsb::launch_project_packed(*opt, N, C, width, height, means, quats, scales, opacities, colors,
                                      opt->sh_degree >= 0 ? K : 1, viewmats, Ks, nnz_capacity, nnz, overflow,
                                      camera_ids, gaussian_ids, radii, splats, workspace,
                                      static_cast<cudaStream_t>(stream));
}

size_t gs_isect_packed_workspace_size(int32_t C, int64_t nnz_capacity, int32_t width, int32_t height,
                                      int64_t M_capacity) {
    if (C < 1 || nnz_capacity < 0 || width < 1 || height < 1 || M_capacity < 0) return 0;
    return gsb::isect_workspace_bytes(nnz_capacity, M_capacity);
}

gs_status gs_isect_tiles_packed(const gs_options* opt, int32_t C, int64_t nnz_capacity, const int64_t* nnz,
                                int32_t width, int32_t height, const int32_t* camera_ids, const int32_t* radii,
                                const float* splats, int64_t M_capacity, int64_t* M, int32_t* overflow,
                                int32_t* isect_ids, uint64_t* isect_keys, int32_t* tile_offsets, void* workspace,
                                size_t workspace_bytes, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 1);
    GS_TRY(check_dims(nnz_capacity, 1, width, height));
    GS_TRY(check_dims(0, C, width, height));
    GS_REQ(M_capacity >= 0 && M_capacity < ((int64_t)1 << 31) - 1);
    GS_REQ(nnz && M && overflow && tile_offsets && workspace);
    GS_REQ(nnz_capacity == 0 || (camera_ids && radii && splats));
    GS_REQ(M_capacity == 0 || isect_ids);
    GS_REQ(aligned8(nnz) && aligned8(M) && aligned4(overflow) && aligned4(tile_offsets) && aligned4(isect_ids) &&
           aligned8(isect_keys) && aligned4(camera_ids) && aligned8(radii) && aligned16(splats) &&
           (reinterpret_cast<uintptr_t>(workspace) & 255u) == 0);
    GS_REQ(workspace_bytes >= gsb::isect_workspace_bytes(nnz_capacity, M_capacity));
    return gsb::launch_isect(*opt, C, 0, width, height, radii, splats, nnz_capacity, nnz, camera_ids, M_capacity, M,
                             overflow, isect_ids, isect_keys, tile_offsets, workspace, workspace_bytes,
                             static_cast<cudaStream_t>(stream));
}

size_t gs_project_bwd_packed_workspace_size(int64_t N, int32_t C) {
    if (N < 0 || C < 1) return 0;
    return gsb::project_bwd_packed_workspace_bytes(N, C);
}

gs_status gs_project_bwd_packed(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                                const float* means, const float* quats, const float* scales, const float* opacities,
                                const float* colors, int32_t K, const float* viewmats, const float* Ks,
                                int64_t nnz_capacity, const int64_t* nnz, const int32_t* camera_ids,
                                const int32_t* gaussian_ids, const int32_t* radii, const float* v_splats,
                                float* v_means, float* v_quats, float* v_scales, float* v_opacities, float* v_colors,
                                float* v_viewmats, void* workspace, size_t workspace_bytes, void* stream) {
    GS_TRY(check_opts(opt));
    GS_REQ(opt->packed == 1);
    GS_TRY(check_raster_dims(opt, N, C, width, height));   // packed: item ids < 2^31, not C*N
    GS_REQ(aligned4(v_viewmats));
    if (N == 0)
        return gsb::launch_project_bwd_packed(*opt, 0, C, width, height, nullptr, nullptr, nullptr, nullptr, nullptr, 1,
                                              nullptr, nullptr, 0, nnz, nullptr, nullptr, nullptr, nullptr, nullptr,
                                              nullptr, nullptr, nullptr, nullptr, v_viewmats, nullptr,
                                              static_cast<cudaStream_t>(stream));
    GS_REQ(nnz_capacity >= 0 && nnz && workspace && (reinterpret_cast<uintptr_t>(workspace) & 255u) == 0);
    GS_REQ(workspace_bytes >= gsb::project_bwd_packed_workspace_bytes(N, C));
    GS_REQ(means && quats && scales && opacities && viewmats && Ks && v_means && v_quats && v_scales &&
           v_opacities && (opt->sh_degree < 0 || (colors && v_colors)));
    GS_REQ(nnz_capacity == 0 || (camera_ids && gaussian_ids && radii && v_splats));
    GS_REQ(aligned8(nnz) && aligned16(quats) && aligned16(v_quats) && aligned16(v_splats) && aligned8(radii) &&
           aligned4(camera_ids) && aligned4(gaussian_ids) && aligned4(means) && aligned4(v_means) &&
           aligned4(colors) && aligned4(v_colors) && aligned4(scales) && aligned4(v_scales));
    if (opt->sh_degree >= 0) GS_REQ(K >= (opt->sh_degree + 1) * (opt->sh_degree + 1));
    return gsb::launch_project_bwd_packed(*opt, N, C, width, height, means, quats, scales, opacities, colors,
                                          opt->sh_degree >= 0 ? K : 1, viewmats, Ks, nnz_capacity, nnz, camera_ids,
                                          gaussian_ids, radii, v_splats, v_means, v_quats, v_scales, v_opacities,
                                          v_colors, v_viewmats, workspace, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
