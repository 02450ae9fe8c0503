// Densification statistics (App. ADC, Absgrad P:204-206):
// per Gaussian, over the cameras where it is visible, the accumulated norm of the
// view-space positional gradient (signed, or the Absgrad per-pixel absolute sums that
// gs_rasterize_bwd writes into v_splats slots 10 and 11), the visible-view count and the
// largest screen radius.  In-place accumulators across calls (training steps).
//
// Dense: one thread per Gaussian sums its C cameras in order (deterministic, no atomics).
// Packed: one thread per visible item, float / int atomics into the per-Gaussian rows.
#include "gs_internal.cuh"

namespace gsb {
namespace {

__device__ __forceinline__ float view_norm(const float* row, int absgrad, float sx, float sy) {
    const float gx = sx * row[absgrad ? 10 : 0], gy = sy * row[absgrad ? 11 : 1];
    return sqrtf(gx * gx + gy * gy);
}

__global__ void k_stats_dense(int64_t N, int C, const int2* __restrict__ radii, const float* __restrict__ v_splats,
                              int absgrad, float sx, float sy, float rscale, float* grad2d, int32_t* count,
                              float* max_radii) {
    pdl_trigger();
    pdl_wait();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    float g = 0.f, mr = 0.f;
    int cnt = 0;
    for (int c = 0; c < C; c++) {
        const int64_t idx = (int64_t)c * N + n;
        const int2 r = radii[idx];
        if (r.x > 0 && r.y > 0) {
            g += view_norm(v_splats + idx * GS_SPLAT_FLOATS, absgrad, sx, sy);
            cnt++;
            mr = fmaxf(mr, (float)max(r.x, r.y) * rscale);
        }
    }
    grad2d[n] += g;
    count[n] += cnt;
    max_radii[n] = fmaxf(max_radii[n], mr);
}

__global__ void k_stats_packed(const int64_t* d_nnz, int64_t cap, const int32_t* __restrict__ gids,
                               const int2* __restrict__ radii, const float* __restrict__ v_splats, int absgrad, float sx,
                               float sy, float rscale, float* grad2d, int32_t* count, float* max_radii) {
    pdl_trigger();
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= min(*d_nnz, cap)) return;
    const int2 r = radii[i];
    if (!(r.x > 0 && r.y > 0)) return;
    const int64_t n = gids[i];
    atomicAdd(grad2d + n, view_norm(v_splats + i * GS_SPLAT_FLOATS, absgrad, sx, sy));
    atomicAdd(count + n, 1);
    // non-negative floats order like their bit patterns
    atomicMax(reinterpret_cast<int*>(max_radii + n), __float_as_int((float)max(r.x, r.y) * rscale));
}

}  // namespace
}  // namespace gsb

using namespace gsb;

extern "C" gs_status gs_densify_stats(const gs_options* opt, int64_t N, int32_t C, int64_t nnz_capacity,
                                      const int64_t* nnz, const int32_t* gaussian_ids, const int32_t* radii,
                                      const float* v_splats, int32_t absgrad, float sx, float sy,
                                      float radius_scale, float* grad2d, int32_t* count, float* max_radii,
                                      void* stream) {
    if (!opt || N < 0 || C < 1 || !(radius_scale >= 0.f)) return GS_ERR_INVALID_ARGUMENT;
    if (N == 0) return GS_OK;
    if (!grad2d || !count || !max_radii || !radii || !v_splats) return GS_ERR_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(radii) & 7u) || (reinterpret_cast<uintptr_t>(v_splats) & 15u))
        return GS_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (opt->packed) {
        if (!nnz || !gaussian_ids || nnz_capacity < 0) return GS_ERR_INVALID_ARGUMENT;
        if (nnz_capacity > 0)
            launch_pdl(k_stats_packed, dim3(div_up(nnz_capacity, 256)), dim3(256), s, nnz, nnz_capacity, gaussian_ids,
                       reinterpret_cast<const int2*>(radii), v_splats, (int)(absgrad != 0), sx, sy, radius_scale,
                       grad2d, count, max_radii);
    } else {
        launch_pdl(k_stats_dense, dim3(div_up(N, 256)), dim3(256), s, N, (int)C, reinterpret_cast<const int2*>(radii),
                   v_splats, (int)(absgrad != 0), sx, sy, radius_scale, grad2d, count, max_radii);
    }
    GS_LAUNCH_CHECK("gs_densify_stats");
    return GS_OK;
}
