// Stage 3 (K6) and stage 4a (K7): per-pixel compositing forward and backward -- R1..R3 and
// B1..B6 of SURVEY Appendix A, restating App. B.2 and App. C.2 of
// arXiv 2409.06765.
//
// Design (B200): one CTA per 16x16 tile, one thread per pixel.  The tile's
// depth-sorted range is walked in batches of 256 splats; each batch is gathered from the
// 48-byte projected records (L2-resident at 1-MP scale) into shared memory once and then
// broadcast to all 256 pixels (TMA-free on purpose: the gather is an indirect load through
// isect_ids, which cp.async.bulk cannot express).  The conic is pre-scaled by -log2(e) at
// staging so the per-pair exponent is two FMAs and one MUFU.EX2.  Forward and backward
// evaluate alpha with the SAME inline function built from _rn intrinsics, so the skip
// decisions of the backward replay those of the forward bit for bit.  The backward reduces
// each splat's 9 gradient values across the warp with shuffles and issues three 16-byte
// vector reductions (red.global.add.v4.f32) per (splat, warp) that touched it.
// These kernels are bound by FP32/MUFU issue, not HBM (DESIGN.md roofline K6/K7).
#include "gs_internal.cuh"

namespace gsb {
namespace {

constexpr int kBatch = GS_BLOCK_PIXELS;   // 256 splats per staged batch
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Pre-scaled conic: p = a' dx^2 + c' dy^2 + b' dx dy = -sigma * log2(e)
__device__ __forceinline__ float4 prescale_conic(float A, float B, float C) {
    return make_float4(__fmul_rn(-0.5f * kLog2e, A), __fmul_rn(-kLog2e, B), __fmul_rn(-0.5f * kLog2e, C), 0.f);
}

// alpha of one (pixel, splat) pair; returns false when the pair is skipped (sigma < 0 or
// alpha < alpha_min, Q14).  G = exp(-sigma).  Bit-identical in K6 and K7.
__device__ __forceinline__ bool eval_alpha(float mx, float my, float o, float4 con, float fpx, float fpy,
                                           float alpha_max, float alpha_min, float& dx, float& dy, float& G,
                                           float& alpha) {
    dx = __fsub_rn(mx, fpx);   // Delta = mu' - p (Q21)
    dy = __fsub_rn(my, fpy);
    const float p = __fmaf_rn(con.y, __fmul_rn(dx, dy),
                              __fmaf_rn(con.x, __fmul_rn(dx, dx), __fmul_rn(con.z, __fmul_rn(dy, dy))));
    if (p > 0.f) return false;   // sigma < 0
    G = ex2_approx(p);
    alpha = fminf(alpha_max, __fmul_rn(o, G));
    return alpha >= alpha_min;
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

struct RasterParams {
    int C, W, H, TX, TY;
    int64_t N;
    float alpha_max, alpha_min, t_min;
    const float* splats;
    const float* bg;
    const int32_t* ids;
    const int32_t* offs;
    float* out_rgb;
    float* out_alpha;
    float* out_T;
    int32_t* last_ids;
    // backward
    const float* v_rgb;
    const float* v_alpha;
    float* v_splats;
    int absgrad;
    // diagnostics (gs_rasterize_stats)
    int32_t* n_eval;
    int32_t* n_contrib;
};

template <bool STATS>
__global__ void __launch_bounds__(kBatch) k_raster_fwd(RasterParams p) {
    __shared__ float4 s_xyo[kBatch];
    __shared__ float4 s_con[kBatch];
    __shared__ float4 s_rgb[kBatch];
    const int tile = blockIdx.x, cam = blockIdx.y;
    const int tx = tile % p.TX, ty = tile / p.TX;
    const int px = tx * GS_TILE + (threadIdx.x & (GS_TILE - 1));
    const int py = ty * GS_TILE + (threadIdx.x / GS_TILE);
    const bool inside = px < p.W && py < p.H;
    const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;   // pixel centre
    const int bin = cam * p.TX * p.TY + tile;
    const int start = p.offs[bin], end = p.offs[bin + 1];

    float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
    int last = start - 1;
    bool done = !inside;
    int n_eval = 0, n_contrib = 0;
    for (int b0 = start; b0 < end; b0 += kBatch) {
        if (__syncthreads_count(done) == kBatch) break;
        const int idx = b0 + threadIdx.x;
        if (idx < end) {
            const int64_t g = p.ids[idx];
            const float4* rec = reinterpret_cast<const float4*>(p.splats + g * GS_SPLAT_FLOATS);
            const float4 r0 = __ldg(rec), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2);
            s_xyo[threadIdx.x] = r0;
            s_con[threadIdx.x] = prescale_conic(r1.x, r1.y, r1.z);
            s_rgb[threadIdx.x] = r2;
        }
        __syncthreads();
        if (!done) {
            const int n = min(kBatch, end - b0);
            for (int j = 0; j < n; j++) {
                const float4 xyo = s_xyo[j];
                float dx, dy, G, alpha;
                if (STATS) n_eval++;
                if (!eval_alpha(xyo.x, xyo.y, xyo.z, s_con[j], fpx, fpy, p.alpha_max, p.alpha_min, dx, dy, G, alpha))
                    continue;
                const float nT = __fmul_rn(T, __fsub_rn(1.f, alpha));
                if (nT <= p.t_min) {   // Q15: stop without compositing this splat
                    done = true;
                    break;
                }
                const float w = __fmul_rn(alpha, T);
                const float4 rgb = s_rgb[j];
                c0 = __fmaf_rn(rgb.x, w, c0);   // C += c alpha T
                c1 = __fmaf_rn(rgb.y, w, c1);
                c2 = __fmaf_rn(rgb.z, w, c2);
                T = nT;
                last = b0 + j;
                if (STATS) n_contrib++;
            }
        }
    }
    if (STATS) {
        if (inside) {
            const int64_t pix = ((int64_t)cam * p.H + py) * p.W + px;
            p.n_eval[pix] = n_eval;
            p.n_contrib[pix] = n_contrib;
        }
        return;
    }
    if (inside) {
        const int64_t pix = ((int64_t)cam * p.H + py) * p.W + px;
        float b0 = 0.f, b1 = 0.f, b2 = 0.f;
        if (p.bg) {
            b0 = p.bg[3 * cam];
            b1 = p.bg[3 * cam + 1];
            b2 = p.bg[3 * cam + 2];
        }
        p.out_rgb[3 * pix + 0] = c0 + T * b0;   // R3, Q25
        p.out_rgb[3 * pix + 1] = c1 + T * b1;
        p.out_rgb[3 * pix + 2] = c2 + T * b2;
        p.out_alpha[pix] = 1.f - T;
        p.out_T[pix] = T;
        p.last_ids[pix] = last;
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <bool ABSGRAD>
__global__ void __launch_bounds__(kBatch) k_raster_bwd(RasterParams p) {
    __shared__ float4 s_xyo[kBatch];
    __shared__ float4 s_con[kBatch];
    __shared__ float4 s_rgb[kBatch];
    __shared__ int32_t s_id[kBatch];
    __shared__ int s_maxlast;
    const int tile = blockIdx.x, cam = blockIdx.y;
    const int tx = tile % p.TX, ty = tile / p.TX;
    const int px = tx * GS_TILE + (threadIdx.x & (GS_TILE - 1));
    const int py = ty * GS_TILE + (threadIdx.x / GS_TILE);
    const bool inside = px < p.W && py < p.H;
    const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;
    const int bin = cam * p.TX * p.TY + tile;
    const int start = p.offs[bin];
    const int lane = threadIdx.x & 31;

    float Tfin = 1.f, v0 = 0.f, v1 = 0.f, v2 = 0.f, vA = 0.f, bgdot = 0.f;
    int last = start - 1;
    if (inside) {
        const int64_t pix = ((int64_t)cam * p.H + py) * p.W + px;
        Tfin = p.out_T[pix];
        last = p.last_ids[pix];
        v0 = p.v_rgb[3 * pix + 0];
        v1 = p.v_rgb[3 * pix + 1];
        v2 = p.v_rgb[3 * pix + 2];
        if (p.v_alpha) vA = p.v_alpha[pix];
        if (p.bg) bgdot = p.bg[3 * cam] * v0 + p.bg[3 * cam + 1] * v1 + p.bg[3 * cam + 2] * v2;
    }
    if (threadIdx.x == 0) s_maxlast = start - 1;
    __syncthreads();
    {
        int m = __reduce_max_sync(0xffffffffu, last);
        if (lane == 0) atomicMax(&s_maxlast, m);
    }
    __syncthreads();
    const int max_last = s_maxlast;
    // constant part of d C_total / d alpha_k: -T_final ra (bg . v_C) + T_final ra v_A (B4)
    const float kbg = Tfin * (vA - bgdot);

    float T = Tfin, S0 = 0.f, S1 = 0.f, S2 = 0.f;
    for (int bend = max_last + 1; bend > start; bend -= kBatch) {
        const int bstart = max(start, bend - kBatch);
        __syncthreads();
        const int idx = bstart + threadIdx.x;
        if (idx < bend) {
            const int32_t g = p.ids[idx];
            const float4* rec = reinterpret_cast<const float4*>(p.splats + (int64_t)g * GS_SPLAT_FLOATS);
            const float4 r0 = __ldg(rec), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2);
            s_xyo[threadIdx.x] = r0;
            s_con[threadIdx.x] = prescale_conic(r1.x, r1.y, r1.z);
            s_rgb[threadIdx.x] = r2;
            s_id[threadIdx.x] = g;
        }
        __syncthreads();
        for (int j = bend - 1 - bstart; j >= 0; j--) {
            const int k = bstart + j;
            bool valid = inside && k <= last;
            const float4 xyo = s_xyo[j];
            const float4 con = s_con[j];
            float dx = 0.f, dy = 0.f, G = 0.f, alpha = 0.f;
            if (valid)
                valid = eval_alpha(xyo.x, xyo.y, xyo.z, con, fpx, fpy, p.alpha_max, p.alpha_min, dx, dy, G, alpha);
            if (!__any_sync(0xffffffffu, valid)) continue;
            float g_mx = 0.f, g_my = 0.f, g_o = 0.f, g_a = 0.f, g_b = 0.f, g_c = 0.f, g_r = 0.f, g_g = 0.f, g_bl = 0.f;
            if (valid) {
                const float4 rgb = s_rgb[j];
                const float ra = 1.f / (1.f - alpha);
                T = T * ra;                        // B2: T_{n-1} = T_n / (1 - alpha_{n-1})
                const float fac = alpha * T;
                g_r = fac * v0;                    // B3
                g_g = fac * v1;
                g_bl = fac * v2;
                // B4 + background / alpha-output terms (Q25, Q26)
                const float v_alpha = (rgb.x * T - S0 * ra) * v0 + (rgb.y * T - S1 * ra) * v1 +
                                      (rgb.z * T - S2 * ra) * v2 + kbg * ra;
                S0 += rgb.x * fac;                 // B5
                S1 += rgb.y * fac;
                S2 += rgb.z * fac;
                const float raw = xyo.z * G;
                if (raw < p.alpha_max) {           // B6 (Q24)
                    g_o = G * v_alpha;
                    const float v_sigma = -raw * v_alpha;
                    g_a = 0.5f * v_sigma * dx * dx;
                    g_b = v_sigma * dx * dy;
                    g_c = 0.5f * v_sigma * dy * dy;
                    // d sigma / d mu' = Sigma'^-1 Delta, with the conic recovered from
                    // the pre-scaled one: A = a' (-2 ln2), B = b' (-ln2), C = c' (-2 ln2)
                    const float k2 = -kLn2 * v_sigma;
                    g_mx = k2 * (2.f * con.x * dx + con.y * dy);
                    g_my = k2 * (con.y * dx + 2.f * con.z * dy);
                }
            }
            float a_mx = 0.f, a_my = 0.f;
            if (ABSGRAD) {
                a_mx = warp_sum(fabsf(g_mx));
                a_my = warp_sum(fabsf(g_my));
            }
            g_mx = warp_sum(g_mx);
            g_my = warp_sum(g_my);
            g_o = warp_sum(g_o);
            g_a = warp_sum(g_a);
            g_b = warp_sum(g_b);
            g_c = warp_sum(g_c);
            g_r = warp_sum(g_r);
            g_g = warp_sum(g_g);
            g_bl = warp_sum(g_bl);
            if (lane == 0) {
                float* dst = p.v_splats + (int64_t)s_id[j] * GS_SPLAT_FLOATS;
                red_add_v4(dst, g_mx, g_my, g_o, 0.f);
                red_add_v4(dst + 4, g_a, g_b, g_c, a_mx);
                red_add_v4(dst + 8, g_r, g_g, g_bl, a_my);
            }
        }
    }
}

RasterParams make_params(const gs_options& o, int C, int64_t N, int W, int H, const float* splats, const float* bg,
                         const int32_t* ids, const int32_t* offs) {
    RasterParams p{};
    p.C = C; p.W = W; p.H = H; p.N = N;
    p.TX = div_up(W, GS_TILE); p.TY = div_up(H, GS_TILE);
    p.alpha_max = o.alpha_max; p.alpha_min = o.alpha_min; p.t_min = o.t_min;
    p.splats = splats; p.bg = bg; p.ids = ids; p.offs = offs;
    return p;
}

}  // namespace

gs_status launch_raster_fwd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats, const float* bg,
                            const int32_t* ids, const int32_t* offs, float* out_rgb, float* out_alpha, float* out_T,
                            int32_t* last_ids, cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, bg, ids, offs);
    p.out_rgb = out_rgb; p.out_alpha = out_alpha; p.out_T = out_T; p.last_ids = last_ids;
    dim3 grid(p.TX * p.TY, C);
    k_raster_fwd<false><<<grid, kBatch, 0, s>>>(p);
    GS_LAUNCH_CHECK("k_raster_fwd");
    return GS_OK;
}

gs_status launch_raster_stats(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                              const int32_t* ids, const int32_t* offs, int32_t* n_eval, int32_t* n_contrib,
                              cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, nullptr, ids, offs);
    p.n_eval = n_eval; p.n_contrib = n_contrib;
    dim3 grid(p.TX * p.TY, C);
    k_raster_fwd<true><<<grid, kBatch, 0, s>>>(p);
    GS_LAUNCH_CHECK("k_raster_fwd<stats>");
    return GS_OK;
}

gs_status launch_raster_bwd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats, const float* bg,
                            const int32_t* ids, const int32_t* offs, const float* out_T, const int32_t* last_ids,
                            const float* v_rgb, const float* v_alpha, int absgrad, float* v_splats, cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, bg, ids, offs);
    p.out_T = const_cast<float*>(out_T); p.last_ids = const_cast<int32_t*>(last_ids);
    p.v_rgb = v_rgb; p.v_alpha = v_alpha; p.v_splats = v_splats; p.absgrad = absgrad;
    if (N > 0 && cudaMemsetAsync(v_splats, 0, sizeof(float) * GS_SPLAT_FLOATS * (size_t)C * (size_t)N, s) != cudaSuccess) {
        GS_LAUNCH_CHECK("v_splats memset");
        return GS_ERR_CUDA;
    }
    dim3 grid(p.TX * p.TY, C);
    if (absgrad)
        k_raster_bwd<true><<<grid, kBatch, 0, s>>>(p);
    else
        k_raster_bwd<false><<<grid, kBatch, 0, s>>>(p);
    GS_LAUNCH_CHECK("k_raster_bwd");
    return GS_OK;
}

}  // namespace gsb
