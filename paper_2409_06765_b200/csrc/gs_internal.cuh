// Internal declarations shared by the sm_100a kernels of libgsplat_b200.
// (The oracle in /oracle shares nothing with this file.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gs.h"

#define GS_TILE 16
#define GS_BLOCK_PIXELS (GS_TILE * GS_TILE)

// Launch-error capture: returns GS_ERR_CUDA from the enclosing gs_status function.
namespace gsb {
void set_last_error(const char* where, cudaError_t e);
}
#define GS_LAUNCH_CHECK(where)                                   \
    do {                                                         \
        cudaError_t e_ = cudaGetLastError();                     \
        if (e_ != cudaSuccess) {                                 \
            gsb::set_last_error(where, e_);                      \
            return GS_ERR_CUDA;                                  \
        }                                                        \
    } while (0)

namespace gsb {

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl() may be
// scheduled while its predecessor in the stream is still running; it calls pdl_trigger()
// (let ITS successor launch early) and pdl_wait() (block until the predecessor grid has
// completed and its memory is visible) before touching anything the predecessor wrote.
// This hides the launch / ramp-up latency of the many short kernels of stage 2.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__host__ __device__ inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

inline int tile_bits(int ntiles) {
    int B = 0;
    while ((1LL << B) < ntiles) B++;
    return B;
}

// ---- stage launchers (defined in project.cu / isect.cu / raster.cu) ----
gs_status launch_project_fwd(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                             const float* quats, const float* scales, const float* opac,
                             const float* colors, int K, const float* viewmats, const float* Ks,
                             int32_t* radii, float* splats, cudaStream_t s);
gs_status launch_project_bwd(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                             const float* quats, const float* scales, const float* opac,
                             const float* colors, int K, const float* viewmats, const float* Ks,
                             const int32_t* radii, const float* v_splats, float* v_means,
                             float* v_quats, float* v_scales, float* v_opac, float* v_colors,
                             float* v_viewmats, void* ws, cudaStream_t s);
size_t project_bwd_workspace_bytes(int64_t N, int C);
size_t project_packed_workspace_bytes(int64_t N, int C);
gs_status launch_project_packed(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                                const float* quats, const float* scales, const float* opac, const float* colors,
                                int K, const float* viewmats, const float* Ks, int64_t cap, int64_t* nnz,
                                int32_t* overflow, int32_t* camera_ids, int32_t* gaussian_ids, int32_t* radii,
                                float* splats, void* ws, cudaStream_t s);
size_t project_bwd_packed_workspace_bytes(int64_t N, int C);
gs_status launch_project_bwd_range(const gs_options& o, int64_t N, int64_t n_begin, int64_t n_end, int C, int W,
                                   int H, const float* means, const float* quats, const float* scales,
                                   const float* opac, const float* colors, int K, const float* viewmats,
                                   const float* Ks, const int32_t* radii, const float* v_splats, float* v_means,
                                   float* v_quats, float* v_scales, float* v_opac, float* v_colors, cudaStream_t s);
gs_status launch_project_bwd_packed(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                                    const float* quats, const float* scales, const float* opac,
                                    const float* colors, int K, const float* viewmats, const float* Ks,
                                    int64_t cap, const int64_t* nnz, const int32_t* camera_ids,
                                    const int32_t* gaussian_ids, const int32_t* radii, const float* v_splats,
                                    float* v_means, float* v_quats, float* v_scales, float* v_opac,
                                    float* v_colors, float* v_viewmats, void* ws, cudaStream_t s);
// n_items = C*N dense items (camera = id / N), or the packed capacity with the live count
// *d_nnz and camera_ids (both NULL in dense mode).
size_t isect_workspace_bytes(int64_t n_items, int64_t cap);
gs_status launch_isect(const gs_options& o, int C, int64_t N, int W, int H, const int32_t* radii,
                       const float* splats, int64_t n_items, const int64_t* d_nnz, const int32_t* camera_ids,
                       int64_t cap, int64_t* M, int32_t* overflow, int32_t* ids, uint64_t* keys,
                       int32_t* tile_offsets, void* ws, size_t ws_bytes, cudaStream_t s);
gs_status launch_raster_fwd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                            const float* bg, const int32_t* ids, const int32_t* offs, float* out_rgb,
                            float* out_alpha, float* out_T, int32_t* last_ids, float* out_depth, int depth_mode,
                            uint16_t* isect_masks, cudaStream_t s);
gs_status launch_raster_stats(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                              const int32_t* ids, const int32_t* offs, int32_t* n_eval, int32_t* n_contrib,
                              int32_t* terminated, cudaStream_t s);
gs_status launch_raster_bwd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                            const float* bg, const int32_t* ids, const int32_t* offs, const float* out_T,
                            const int32_t* last_ids, const float* v_rgb, const float* v_alpha,
                            const float* out_depth, const float* v_depth, int depth_mode, int absgrad,
                            const uint16_t* isect_masks, const int32_t* tile_order, float* v_splats,
                            cudaStream_t s);
gs_status launch_tile_order(int C, int W, int H, const int32_t* offs, int32_t* order, cudaStream_t s);
gs_status launch_zero_splat_grads(float* v_splats, size_t nrec, cudaStream_t s);
gs_status launch_raster_fwd_nd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                               const float* feats, int D, const int32_t* gids, const float* bg, const int32_t* ids,
                               const int32_t* offs, float* out_feats, float* out_alpha, float* out_T,
                               int32_t* last_ids, uint16_t* isect_masks, cudaStream_t s);
gs_status launch_raster_bwd_nd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                               const float* feats, int D, const int32_t* gids, int64_t n_gauss, const float* bg,
                               const int32_t* ids, const int32_t* offs, const float* out_T, const int32_t* last_ids,
                               const float* v_feats_img, const float* v_alpha, int absgrad,
                               const uint16_t* isect_masks, float* v_splats, float* v_feats, cudaStream_t s);

}  // namespace gsb
