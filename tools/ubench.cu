// Microbenchmarks of the units the raster kernels are bound by ("a
// microbenchmark for FP32 FMA, MUFU ex2, SHFL and RED throughput -- those ALU roofs are not
// measured in MP").  Standalone: `python tools/ubench.py` builds it for sm_100a and writes
// the JSON it prints to profiles/.  Each kernel runs a fixed instruction count on a grid of
// 148 SMs x 8 CTAs x 256 threads; rates are thread-instructions (or operations) per second,
// timed with CUDA events after a warm-up launch.
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            return 1;                                                          \
        }                                                                      \
    } while (0)

constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 1.2345f) out[0] = s;
}

__global__ void k_ex2(float* out, float a) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = -1e-3f * (threadIdx.x + i);
    for (int it = 0; it < kIters / 4; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
            x[i] = y * a;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 1.2345f) out[0] = s;
}

__global__ void k_shfl(float* out) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
    for (int it = 0; it < kIters / 4; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 << (i & 3));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 1.2345f) out[0] = s;
}

__global__ void k_lds128(float* out) {
    __shared__ float4 sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int idx = threadIdx.x;
    for (int it = 0; it < kIters / 4; it++) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float4 v = sm[(idx + 32 * i) & 1023];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        idx += 7;
    }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;
}

// red.global.add.v4.f32: `lanes` active lanes per warp all hitting ONE 16-byte address per
// warp-iteration (the few-lanes path of K7: every contributing lane reduces into the same
// splat record), addresses spread over a 48 MB table like K7's v_splats.
__global__ void k_red_v4_same(float* table, int lanes, int n_rows) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane >= lanes) return;
    unsigned h = warp * 2654435761u;
    for (int it = 0; it < kIters / 16; it++) {
        h = h * 1664525u + 1013904223u;
        float* dst = table + (size_t)(h % (unsigned)n_rows) * 12;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
    }
}

// scalar red.global.add.f32, one address per lane (the tree path: 8-9 lanes, distinct slots)
__global__ void k_red_f32_distinct(float* table, int n_rows) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned h = warp * 2654435761u;
    for (int it = 0; it < kIters / 16; it++) {
        h = h * 1664525u + 1013904223u;
        float* dst = table + (size_t)(h % (unsigned)n_rows) * 12 + (lane % 12);
        atomicAdd(dst, 1.f);
    }
}

// red.global.add.v4.f32, every lane its own random record (no same-address contention)
__global__ void k_red_v4_distinct(float* table, int n_rows) {
    unsigned h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    for (int it = 0; it < kIters / 16; it++) {
        h = h * 1664525u + 1013904223u;
        float* dst = table + (size_t)(h % (unsigned)n_rows) * 12;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
    }
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename F>
float time_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms / 5.f;
}

int main() {
    int sms = 0, clk_khz = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    const dim3 grid(sms * 8), block(256);
    const double threads = (double)grid.x * block.x;
    float* out;
    CK(cudaMalloc(&out, 64));
    const int n_rows = 1000000;   // 48 MB table of 12-float records
    float* table;
    CK(cudaMalloc(&table, (size_t)n_rows * 12 * sizeof(float)));
    CK(cudaMemset(table, 0, (size_t)n_rows * 12 * sizeof(float)));

    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f", sms, clk_khz / 1e3);
    float ms = time_ms([&] { k_ffma<<<grid, block>>>(out, 0.999f, 1e-3f); });
    printf(", \"ffma_T_per_s\": %.3f", threads * kIters * 8 / (ms * 1e-3) / 1e12);
    ms = time_ms([&] { k_ex2<<<grid, block>>>(out, 0.999f); });
    printf(", \"mufu_ex2_T_per_s\": %.3f", threads * (kIters / 4) * 8 / (ms * 1e-3) / 1e12);
    ms = time_ms([&] { k_shfl<<<grid, block>>>(out); });
    printf(", \"shfl_T_per_s\": %.3f", threads * (kIters / 4) * 8 / (ms * 1e-3) / 1e12);
    ms = time_ms([&] { k_lds128<<<grid, block>>>(out); });
    printf(", \"lds128_TB_per_s\": %.3f", threads * (kIters / 4) * 4 * 16 / (ms * 1e-3) / 1e12);
    printf(", \"red_v4_same_address\": {");
    const int lane_counts[] = {1, 2, 4, 8, 16, 32};
    for (int k = 0; k < 6; k++) {
        const int L = lane_counts[k];
        ms = time_ms([&] { k_red_v4_same<<<grid, block>>>(table, L, n_rows); });
        const double warps = threads / 32;
        printf("%s\"%d_lanes\": {\"G_warp_instr_per_s\": %.2f, \"G_lane_ops_per_s\": %.2f}", k ? ", " : "", L,
               warps * (kIters / 16) / (ms * 1e-3) / 1e9, warps * L * (kIters / 16) / (ms * 1e-3) / 1e9);
    }
    printf("}");
    ms = time_ms([&] { k_red_v4_distinct<<<grid, block>>>(table, n_rows); });
    printf(", \"red_v4_distinct_G_lane_ops_per_s\": %.2f", threads * (kIters / 16) / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { k_red_f32_distinct<<<grid, block>>>(table, n_rows); });
    printf(", \"red_f32_G_lane_ops_per_s\": %.2f", threads * (kIters / 16) / (ms * 1e-3) / 1e9);
    const size_t n4 = (size_t)1 << 26;   // 1 GiB per buffer
    float4 *a, *b;
    CK(cudaMalloc(&a, n4 * 16));
    CK(cudaMalloc(&b, n4 * 16));
    CK(cudaMemset(a, 0, n4 * 16));
    ms = time_ms([&] { k_copy<<<sms * 8, 512>>>(a, b, n4); });
    printf(", \"copy_GB_per_s\": %.1f}\n", 2.0 * n4 * 16 / (ms * 1e-3) / 1e9);
    CK(cudaGetLastError());
    return 0;
}
