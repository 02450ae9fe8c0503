// Gaussian-sharded scale-out: the row packing on either side
// of the two NCCL all-to-alls that move projected records from the Gaussians' owners to
// the views' renderers (and their gradients back).  include/gs.h documents the protocol.
//
// Pure data movement (HBM-bound): one 64-byte row per visible (camera, Gaussian) item,
// written / read as four 16-byte vectors by consecutive threads (fully coalesced).
#include "gs_internal.cuh"

namespace gsb {
namespace {

constexpr int kMaxRanks = 64;

struct ViewStarts {
    int32_t v[kMaxRanks + 1];
};

// Destination rank of camera c: the q with view_starts[q] <= c < view_starts[q+1].
__device__ __forceinline__ int dest_of(const ViewStarts& vs, int R, int c) {
    int lo = 0, hi = R - 1;
    while (lo < hi) {   // last q with v[q] <= c
        const int mid = (lo + hi + 1) >> 1;
        if (vs.v[mid] <= c) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Rows per destination: items are camera-major, so destination q holds the contiguous
// range [lower_bound(view_starts[q]), lower_bound(view_starts[q+1])) of camera_ids.
__global__ void k_shard_counts(const int32_t* __restrict__ cam, const int64_t* d_nnz, int64_t cap, int R,
                               ViewStarts vs, int64_t* __restrict__ counts) {
    pdl_trigger();
    pdl_wait();
    const int q = threadIdx.x;
    if (q >= R) return;
    const int64_t n = min(*d_nnz, cap);
    auto lower = [&](int c) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cam[mid] < c) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    counts[q] = lower(vs.v[q + 1]) - lower(vs.v[q]);
}

__global__ void k_shard_pack(const int32_t* __restrict__ cam, const int64_t* d_nnz, int64_t cap, int R, ViewStarts vs,
                             const int2* __restrict__ radii, const float4* __restrict__ splats,
                             float4* __restrict__ send) {
    pdl_trigger();
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = min(*d_nnz, cap);
    if (i >= n) return;
    const int c = cam[i];
    const int q = dest_of(vs, R, c);
    const int2 r = radii[i];
    const float4* src = splats + i * 3;
    float4* dst = send + i * 4;
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
    dst[3] = make_float4(__int_as_float(r.x), __int_as_float(r.y), __int_as_float(c - vs.v[q]), 0.f);
}

__global__ void k_shard_unpack(int64_t n, const float4* __restrict__ recv, int32_t* __restrict__ cam,
                               int2* __restrict__ radii, float4* __restrict__ splats, int64_t* d_nnz) {
    pdl_trigger();
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *d_nnz = n;
    if (i >= n) return;
    const float4* src = recv + i * 4;
    float4* dst = splats + i * 3;
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
    const float4 t = src[3];
    radii[i] = make_int2(__float_as_int(t.x), __float_as_int(t.y));
    cam[i] = __float_as_int(t.z);
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace gsb

using namespace gsb;

extern "C" {

gs_status gs_shard_pack(int64_t cap, const int64_t* nnz, int32_t C, int32_t R, const int32_t* view_starts,
                        const int32_t* camera_ids, const int32_t* radii, const float* splats, float* send,
                        int64_t* send_counts, void* stream) {
    if (cap < 0 || C < 1 || R < 1 || R > kMaxRanks || !view_starts || !nnz || !send_counts)
        return GS_ERR_INVALID_ARGUMENT;
    if (view_starts[0] != 0 || view_starts[R] != C) return GS_ERR_INVALID_ARGUMENT;
    ViewStarts vs{};
    for (int q = 0; q <= R; q++) {
        if (q > 0 && view_starts[q] < view_starts[q - 1]) return GS_ERR_INVALID_ARGUMENT;
        vs.v[q] = view_starts[q];
    }
    if (cap > 0 && (!camera_ids || !radii || !splats || !send)) return GS_ERR_INVALID_ARGUMENT;
    if (!al16(splats) || !al16(send) || (reinterpret_cast<uintptr_t>(radii) & 7u) ||
        (reinterpret_cast<uintptr_t>(nnz) & 7u) || (reinterpret_cast<uintptr_t>(send_counts) & 7u))
        return GS_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    launch_pdl(k_shard_counts, dim3(1), dim3(kMaxRanks), s, camera_ids, nnz, cap, (int)R, vs, send_counts);
    if (cap > 0)
        launch_pdl(k_shard_pack, dim3(div_up(cap, 256)), dim3(256), s, camera_ids, nnz, cap, (int)R, vs,
                   reinterpret_cast<const int2*>(radii), reinterpret_cast<const float4*>(splats),
                   reinterpret_cast<float4*>(send));
    GS_LAUNCH_CHECK("gs_shard_pack");
    return GS_OK;
}

gs_status gs_shard_unpack(int64_t n_recv, const float* recv, int32_t* camera_ids, int32_t* radii, float* splats,
                          int64_t* nnz, void* stream) {
    if (n_recv < 0 || !nnz) return GS_ERR_INVALID_ARGUMENT;
    if (n_recv > 0 && (!recv || !camera_ids || !radii || !splats)) return GS_ERR_INVALID_ARGUMENT;
    if (!al16(recv) || !al16(splats) || (reinterpret_cast<uintptr_t>(radii) & 7u) ||
        (reinterpret_cast<uintptr_t>(nnz) & 7u))
        return GS_ERR_INVALID_ARGUMENT;
    launch_pdl(k_shard_unpack, dim3(div_up(n_recv > 0 ? n_recv : 1, 256)), dim3(256),
               static_cast<cudaStream_t>(stream), n_recv, reinterpret_cast<const float4*>(recv), camera_ids,
               reinterpret_cast<int2*>(radii), reinterpret_cast<float4*>(splats), nnz);
    GS_LAUNCH_CHECK("gs_shard_unpack");
    return GS_OK;
}

}  // extern "C"
