// Microbenchmark (not product code): staging K6/K7 batches of 48-byte projected records
// into shared memory through the per-tile id lists -- per-thread 16-byte gathers (what the
// raster kernels do) vs TMA tile::gather4 (cp.async.bulk.tensor.2d ... tile::gather4: 4
// rows of a 2D tensor map per instruction, completion on an mbarrier).  Workload shaped like
// BASELINE configs[1]: 1M records, 4346 tiles, 2.87 M ids (random within a tile's list, as
// depth order is unrelated to record order).  Prints the time of one full staging pass each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_gather_ubench tools/tma_gather_ubench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

constexpr int kT = 256, kBatch = 256, kRow = 12;

__global__ void __launch_bounds__(kT) k_threads(const float* __restrict__ rec, const int* __restrict__ ids,
                                                const int* __restrict__ offs, float* out) {
    __shared__ float4 s_a[kBatch], s_b[kBatch], s_c[kBatch];
    const int start = offs[blockIdx.x], end = offs[blockIdx.x + 1];
    float acc = 0.f;
    for (int b0 = start; b0 < end; b0 += kBatch) {
        const int n = min(kBatch, end - b0);
        __syncthreads();
        if ((int)threadIdx.x < n) {
            const float4* r = reinterpret_cast<const float4*>(rec + (size_t)ids[b0 + threadIdx.x] * kRow);
            s_a[threadIdx.x] = __ldg(r);
            s_b[threadIdx.x] = __ldg(r + 1);
            s_c[threadIdx.x] = __ldg(r + 2);
        }
        __syncthreads();
        for (int j = threadIdx.x & 31; j < n; j += 32) acc += s_a[j].x + s_b[j].y + s_c[j].z;
    }
    if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kT) k_tma(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ ids,
                                            const int* __restrict__ offs, float* out) {
    __shared__ alignas(128) float s_rec[kBatch / 4 * 64];   // groups of 4 rows at 256-byte strides
    __shared__ alignas(8) uint64_t mbar;
    const int start = offs[blockIdx.x], end = offs[blockIdx.x + 1];
    const uint32_t bar = smem_u32(&mbar);
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    __syncthreads();
    float acc = 0.f;
    uint32_t phase = 0;
    for (int b0 = start; b0 < end; b0 += kBatch) {
        const int n = min(kBatch, end - b0);
        const int ng = (n + 3) / 4;   // gather4 groups (a ragged tail repeats its last id)
        __syncthreads();              // the previous batch is consumed
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(ng * 4 * kRow * 4));
        __syncthreads();
        if (threadIdx.x < 32) {
            for (int g = threadIdx.x; g < ng; g += 32) {
                int r[4];
#pragma unroll
                for (int k = 0; k < 4; k++) r[k] = ids[b0 + min(4 * g + k, n - 1)];
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(s_rec + g * 64)),
                    "l"(&tmap), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(bar)
                    : "memory");
            }
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar), "r"(phase) : "memory");
        phase ^= 1u;
        for (int j = threadIdx.x & 31; j < n; j += 32) {
            const float* r = s_rec + (j >> 2) * 64 + (j & 3) * kRow;
            acc += r[0] + r[5] + r[10];
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int nrec = 1000000, T = 4346;
    std::mt19937 rng(1);
    std::vector<int> offs(T + 1, 0), ids;
    std::poisson_distribution<int> len(660);
    for (int t = 0; t < T; t++) {
        const int L = len(rng);
        for (int k = 0; k < L; k++) ids.push_back((int)(rng() % nrec));
        offs[t + 1] = (int)ids.size();
    }
    const int M = (int)ids.size();
    float *d_rec, *d_out;
    int *d_ids, *d_offs;
    cudaMalloc(&d_rec, (size_t)nrec * kRow * 4);
    cudaMalloc(&d_ids, (size_t)M * 4);
    cudaMalloc(&d_offs, (T + 1) * 4);
    cudaMalloc(&d_out, 4);
    cudaMemset(d_rec, 0, (size_t)nrec * kRow * 4);
    cudaMemcpy(d_ids, ids.data(), (size_t)M * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_offs, offs.data(), (T + 1) * 4, cudaMemcpyHostToDevice);

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap tmap;
    cuuint64_t dims[2] = {(cuuint64_t)kRow, (cuuint64_t)nrec};
    cuuint64_t strides[1] = {(cuuint64_t)kRow * 4};
    cuuint32_t box[2] = {(cuuint32_t)kRow, 1}, estr[2] = {1, 1};
    CUresult cr = ((EncodeFn)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d_rec, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("{\"error\": \"tensor map %d\"}\n", (int)cr); return 1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms[2];
    for (int v = 0; v < 2; v++) {
        for (int it = 0; it < 3; it++) {
            if (v == 0) k_threads<<<T, kT>>>(d_rec, d_ids, d_offs, d_out);
            else k_tma<<<T, kT>>>(tmap, d_ids, d_offs, d_out);
        }
        cudaEventRecord(a);
        for (int it = 0; it < 20; it++) {
            if (v == 0) k_threads<<<T, kT>>>(d_rec, d_ids, d_offs, d_out);
            else k_tma<<<T, kT>>>(tmap, d_ids, d_offs, d_out);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms[v], a, b);
        ms[v] /= 20;
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"M\": %d, \"records\": %d, \"tiles\": %d, \"threads_ms\": %.4f, \"tma_gather4_ms\": %.4f, \"err\": \"%s\"}\n",
           M, nrec, T, ms[0], ms[1], cudaGetErrorString(e));
    return 0;
}
