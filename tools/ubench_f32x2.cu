// Microbenchmark: sm_100a packed FP32x2 instructions (FFMA2 / FADD2 / FMUL2) against scalar
// FFMA, and whether an FFMA2 frees issue slots for other pipes (the raster kernels K6/K7 are
// issue bound with the FMA pipe ~35 % busy).  Each kernel runs 8 independent
// dependency chains per thread; timings by CUDA events over a grid of 148 x 8 CTAs x 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_f32x2 tools/ubench_f32x2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = __fmaf_rn(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    float2 x[8];
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(x[i], a2, b2);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FFMA2 chains with an independent integer chain interleaved (one LOP3 / IADD per FFMA2)
__global__ void k_ffma2_int(float* out, float a, float b, unsigned m) {
    float2 x[8];
    unsigned u[8];
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; i++) {
        x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        u[i] = threadIdx.x + i;
    }
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            x[i] = __ffma2_rn(x[i], a2, b2);
            u[i] = (u[i] ^ m) + (unsigned)it;
        }
    }
    float s = 0.f;
    unsigned t = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        s += x[i].x + x[i].y;
        t ^= u[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(t & 1u);
}

// scalar FFMA chains with the same integer chain (the reference for the interleaved case)
__global__ void k_ffma_int(float* out, float a, float b, unsigned m) {
    float x[8];
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        x[i] = threadIdx.x * 1e-3f + i;
        u[i] = threadIdx.x + i;
    }
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            x[i] = __fmaf_rn(x[i], a, b);
            u[i] = (u[i] ^ m) + (unsigned)it;
        }
    }
    float s = 0.f;
    unsigned t = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        s += x[i];
        t ^= u[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(t & 1u);
}

int main() {
    const int blocks = 148 * 8, threads = 256;
    float* out;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double warps = (double)blocks * threads / 32.0;
    auto run = [&](const char* name, auto launch, double fma_per_thread_iter, double instr_per_warp_iter) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double s = best / 1e3;
        const double fma = (double)blocks * threads * kIters * fma_per_thread_iter / s;
        const double wi = warps * kIters * instr_per_warp_iter / s;
        printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"T_fp32_lane_ops_per_s\": %.2f, \"G_warp_instr_per_s\": %.1f}\n",
               name, best, fma / 1e12, wi / 1e9);
    };
    run("ffma x8", [&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 8, 8);
    run("ffma2 x8", [&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 16, 8);
    run("ffma x8 + int x8", [&] { k_ffma_int<<<blocks, threads>>>(out, 0.999f, 1e-3f, 0x9e3779b9u); }, 8, 24);
    run("ffma2 x8 + int x8", [&] { k_ffma2_int<<<blocks, threads>>>(out, 0.999f, 1e-3f, 0x9e3779b9u); }, 16, 24);
    cudaDeviceSynchronize();
    return cudaGetLastError() != cudaSuccess;
}
