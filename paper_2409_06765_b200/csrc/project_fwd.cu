// K1: projection of every (camera, Gaussian) -- F1..F15 of SURVEY Appendix A, which
// restates App. B.1 and A.4 of arXiv 2409.06765.
//
// THIS TRANSLATION UNIT IS COMPILED WITH -fmad=false: the fp32 "key path" (t, depth,
// Sigma', radii, mean2d) is evaluated with one IEEE rounding per operator in the fixed
// order written in DESIGN.md (reading Q28), so the tile keys of stage 2 are bit-exact
// functions of the inputs.  The same order is written out, independently, in the oracle.
//
// Design (B200): one thread per Gaussian looping over all cameras of the call, so the
// 44 B of geometry and the up to 192 B of SH coefficients are read from HBM once and
// reused across the C_local views (SH is 81% of the per-Gaussian bytes);
// camera constants live in shared memory; each (c,n) writes one 48 B record as three
// 16 B vector stores plus an 8 B radii store.  HBM-bound (DESIGN.md roofline K1).
#include "gs_internal.cuh"
#include "sh.cuh"

namespace gsb {
namespace {

constexpr int kThreads = 256;
constexpr int kCamChunk = 64;

struct CamConst {
    float vm[12];               // rows 0..2 of the world->camera matrix
    float fx, fy, cx, cy;
    float lxp, lxn, lyp, lyn;   // widened-frustum limits for J (Q27)
    float campos[3];            // -R^T w  (SH view direction)
    float pad;
};

struct ProjParams {
    int64_t N;
    int C, W, H, K;
    float near_plane, far_plane, eps2d, alpha_min;
    int antialiased, bbox_mode, fov_clamp;
    int vec_colors;   // colors base 16B-aligned and K*3 % 4 == 0
    const float* means;
    const float* quats;
    const float* scales;
    const float* opac;
    const float* colors;
    const float* viewmats;
    const float* Ks;
    int32_t* radii;
    float* splats;
    // packed mode (Q29)
    int* blockcnt;            // [C][gridDim.x] visible items per (camera, block); then offsets
    int64_t cap;              // packed capacity
    int32_t* camera_ids;
    int32_t* gaussian_ids;
};

// Kernel modes: dense [C,N] records; packed pass 1 (visibility count per (camera, block));
// packed pass 2 (write each visible record at its packed position).
enum { kDense = 0, kCount = 1, kPacked = 2 };

__device__ __forceinline__ void setup_cam(const ProjParams& p, int c, CamConst& cc) {
    const float* vm = p.viewmats + 16 * (int64_t)c;
    const float* K = p.Ks + 9 * (int64_t)c;
#pragma unroll
    for (int i = 0; i < 12; i++) cc.vm[i] = vm[i];
    cc.fx = K[0];
    cc.fy = K[4];
    cc.cx = K[2];
    cc.cy = K[5];
    float W = (float)p.W, H = (float)p.H;
    float tanx = (0.5f * W) / cc.fx, tany = (0.5f * H) / cc.fy;
    cc.lxp = (W - cc.cx) / cc.fx + 0.3f * tanx;
    cc.lxn = cc.cx / cc.fx + 0.3f * tanx;
    cc.lyp = (H - cc.cy) / cc.fy + 0.3f * tany;
    cc.lyn = cc.cy / cc.fy + 0.3f * tany;
#pragma unroll
    for (int i = 0; i < 3; i++)
        cc.campos[i] = -((vm[0 + i] * vm[3] + vm[4 + i] * vm[7]) + vm[8 + i] * vm[11]);
    cc.pad = 0.f;
}

template <int DEG, int MODE>
__global__ void __launch_bounds__(kThreads) k_project_fwd(ProjParams p) {
    pdl_trigger();
    pdl_wait();
    __shared__ CamConst s_cam[kCamChunk];
    __shared__ int s_wcnt[kThreads / 32];
    const int64_t n = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const bool active = n < p.N;

    // ---- per-Gaussian, camera-independent part of the key path (F1, F2) ----
    float mu0 = 0.f, mu1 = 0.f, mu2 = 0.f, op = 0.f;
    float S00 = 0.f, S01 = 0.f, S02 = 0.f, S10 = 0.f, S11 = 0.f, S12 = 0.f, S20 = 0.f, S21 = 0.f, S22 = 0.f;
    bool qok = false;
    if (active) {
        mu0 = p.means[3 * n + 0];
        mu1 = p.means[3 * n + 1];
        mu2 = p.means[3 * n + 2];
        op = p.opac[n];
        const float4 q = reinterpret_cast<const float4*>(p.quats)[n];
        const float s0 = p.scales[3 * n + 0], s1 = p.scales[3 * n + 1], s2 = p.scales[3 * n + 2];
        // KP3: q_hat = q / ||q||
        float qn2 = ((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w;
        qok = (qn2 > 0.f) && isfinite(qn2);
        float qn = sqrtf(qn2);
        float w = q.x / qn, x = q.y / qn, y = q.z / qn, z = q.w / qn;
        // KP4: R(q_hat)
        float R00 = 1.f - 2.f * (y * y + z * z), R01 = 2.f * (x * y - w * z), R02 = 2.f * (x * z + w * y);
        float R10 = 2.f * (x * y + w * z), R11 = 1.f - 2.f * (x * x + z * z), R12 = 2.f * (y * z - w * x);
        float R20 = 2.f * (x * z - w * y), R21 = 2.f * (y * z + w * x), R22 = 1.f - 2.f * (x * x + y * y);
        // KP5: M = R diag(s); KP6: Sigma = M M^T
        float M00 = R00 * s0, M01 = R01 * s1, M02 = R02 * s2;
        float M10 = R10 * s0, M11 = R11 * s1, M12 = R12 * s2;
        float M20 = R20 * s0, M21 = R21 * s1, M22 = R22 * s2;
        S00 = (M00 * M00 + M01 * M01) + M02 * M02;
        S01 = (M00 * M10 + M01 * M11) + M02 * M12;
        S02 = (M00 * M20 + M01 * M21) + M02 * M22;
        S10 = (M10 * M00 + M11 * M01) + M12 * M02;
        S11 = (M10 * M10 + M11 * M11) + M12 * M12;
        S12 = (M10 * M20 + M11 * M21) + M12 * M22;
        S20 = (M20 * M00 + M21 * M01) + M22 * M02;
        S21 = (M20 * M10 + M21 * M11) + M22 * M12;
        S22 = (M20 * M20 + M21 * M21) + M22 * M22;
    }
    constexpr int NB = DEG < 0 ? 1 : (DEG + 1) * (DEG + 1);

    for (int c0 = 0; c0 < p.C; c0 += kCamChunk) {
        const int nc = min(kCamChunk, p.C - c0);
        __syncthreads();
        if (threadIdx.x < nc) setup_cam(p, c0 + threadIdx.x, s_cam[threadIdx.x]);
        __syncthreads();
        if (MODE == kDense && !active) continue;   // the packed modes keep every thread (block scans)
        for (int ci = 0; ci < nc; ci++) {
            const CamConst& cc = s_cam[ci];
            // KP1 (F3): t = W mu + w
            const float tx = ((cc.vm[0] * mu0 + cc.vm[1] * mu1) + cc.vm[2] * mu2) + cc.vm[3];
            const float ty = ((cc.vm[4] * mu0 + cc.vm[5] * mu1) + cc.vm[6] * mu2) + cc.vm[7];
            const float tz = ((cc.vm[8] * mu0 + cc.vm[9] * mu1) + cc.vm[10] * mu2) + cc.vm[11];
            bool vis = qok && (tz >= p.near_plane) && !(tz > p.far_plane);   // KP2 (F4, Q18)
            float a = 0.f, b = 0.f, c = 0.f, det = 0.f, Sp00 = 0.f, Sp01 = 0.f, Sp11 = 0.f;
            int rx = 0, ry = 0;
            float mx = 0.f, my = 0.f;
            if (vis) {
                // KP7 (F5): Sigma_c = Wr Sigma Wr^T via A = Wr Sigma
                const float* V = cc.vm;
                float A00 = (V[0] * S00 + V[1] * S10) + V[2] * S20;
                float A01 = (V[0] * S01 + V[1] * S11) + V[2] * S21;
                float A02 = (V[0] * S02 + V[1] * S12) + V[2] * S22;
                float A10 = (V[4] * S00 + V[5] * S10) + V[6] * S20;
                float A11 = (V[4] * S01 + V[5] * S11) + V[6] * S21;
                float A12 = (V[4] * S02 + V[5] * S12) + V[6] * S22;
                float A20 = (V[8] * S00 + V[9] * S10) + V[10] * S20;
                float A21 = (V[8] * S01 + V[9] * S11) + V[10] * S21;
                float A22 = (V[8] * S02 + V[9] * S12) + V[10] * S22;
                float C00 = (A00 * V[0] + A01 * V[1]) + A02 * V[2];
                float C01 = (A00 * V[4] + A01 * V[5]) + A02 * V[6];
                float C02 = (A00 * V[8] + A01 * V[9]) + A02 * V[10];
                float C10 = (A10 * V[0] + A11 * V[1]) + A12 * V[2];
                float C11 = (A10 * V[4] + A11 * V[5]) + A12 * V[6];
                float C12 = (A10 * V[8] + A11 * V[9]) + A12 * V[10];
                float C20 = (A20 * V[0] + A21 * V[1]) + A22 * V[2];
                float C21 = (A20 * V[4] + A21 * V[5]) + A22 * V[6];
                float C22 = (A20 * V[8] + A21 * V[9]) + A22 * V[10];
                // KP8 (F6): J with focals (Q4), frustum clamp for J only (Q27)
                float txc = tx, tyc = ty;
                if (p.fov_clamp) {
                    float u = tx / tz, v = ty / tz;
                    float uc = fminf(cc.lxp, fmaxf(-cc.lxn, u)), vc = fminf(cc.lyp, fmaxf(-cc.lyn, v));
                    txc = tz * uc;
                    tyc = tz * vc;
                }
                const float J00 = cc.fx / tz, J01 = 0.f, J02 = -(cc.fx * txc) / (tz * tz);
                const float J10 = 0.f, J11 = cc.fy / tz, J12 = -(cc.fy * tyc) / (tz * tz);
                // KP9 (F7): Sigma' = J Sigma_c J^T via B = J Sigma_c
                float B00 = (J00 * C00 + J01 * C10) + J02 * C20;
                float B01 = (J00 * C01 + J01 * C11) + J02 * C21;
                float B02 = (J00 * C02 + J01 * C12) + J02 * C22;
                float B10 = (J10 * C00 + J11 * C10) + J12 * C20;
                float B11 = (J10 * C01 + J11 * C11) + J12 * C21;
                float B12 = (J10 * C02 + J11 * C12) + J12 * C22;
                Sp00 = (B00 * J00 + B01 * J01) + B02 * J02;
                Sp01 = (B00 * J10 + B01 * J11) + B02 * J12;
                Sp11 = (B10 * J10 + B11 * J11) + B12 * J12;
                // KP10 (F8): low-pass, both modes (Q6)
                a = Sp00 + p.eps2d;
                b = Sp01;
                c = Sp11 + p.eps2d;
                det = a * c - b * b;                                   // KP11 (F9)
                vis = det > 0.f;
                if (vis) {
                    if (p.bbox_mode != 1) {                           // KP12 (F12, Q12)
                        rx = (int)ceilf(3.f * sqrtf(a));
                        ry = (int)ceilf(3.f * sqrtf(c));
                        if (p.bbox_mode == 2 && p.alpha_min > 0.f) {
                            // KP12b (NEXT-4(ii), Q36): opacity-aware extent.  alpha >= alpha_min
                            // needs sigma <= tau = ln(o_eff / alpha_min); tau_ub >= tau from
                            // frexp (x = m 2^e) and ln m <= 2(m-1)/(m+1) on (0, 1].
                            float comp2 = 1.f;
                            if (p.antialiased) {
                                const float det_raw = Sp00 * Sp11 - Sp01 * Sp01;
                                comp2 = sqrtf(fmaxf(0.f, det_raw / det));
                            }
                            const float oe = op * comp2;
                            if (!(oe >= p.alpha_min)) {
                                vis = false;                              // never composited
                            } else {
                                int e2;
                                const float m2 = frexpf(oe / p.alpha_min, &e2);
                                const float tau = (float)e2 * 0.693147182f + (2.f * (m2 - 1.f)) / (m2 + 1.f);
                                const float k2 = 2.f * (tau * 1.004f + 4e-3f);
                                if (k2 < 9.f && (a * c) / det <= 1000.f) {
                                    rx = (int)ceilf(sqrtf(k2 * a));
                                    ry = (int)ceilf(sqrtf(k2 * c));
                                }
                            }
                        }
                    } else {
                        float m = 0.5f * (a + c);
                        float lam = m + sqrtf(fmaxf(0.f, m * m - det));
                        rx = ry = (int)ceilf(3.f * sqrtf(lam));
                    }
                    mx = (cc.fx * tx) / tz + cc.cx;                   // KP13 (F11)
                    my = (cc.fy * ty) / tz + cc.cy;
                    // KP14 (F13, Q19): off-screen cull
                    if (mx + (float)rx <= 0.f || mx - (float)rx >= (float)p.W || my + (float)ry <= 0.f ||
                        my - (float)ry >= (float)p.H || !isfinite(mx) || !isfinite(my))
                        vis = false;
                }
            }
            // ---- where this (c,n) goes ----
            int64_t idx = (int64_t)(c0 + ci) * p.N + n;
            if (MODE == kCount) {
                const int cnt = __syncthreads_count(vis);
                if (threadIdx.x == 0) p.blockcnt[(int64_t)(c0 + ci) * gridDim.x + blockIdx.x] = cnt;
                continue;
            }
            if (MODE == kPacked) {
                // packed position = block offset of camera c + rank of this thread's visible
                // item inside the block (camera-major, then n: Q29)
                const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
                const unsigned bal = __ballot_sync(0xffffffffu, vis);
                __syncthreads();   // s_wcnt reuse across cameras
                if (lane == 0) s_wcnt[warp] = __popc(bal);
                __syncthreads();
                int before = 0;
                for (int w = 0; w < warp; w++) before += s_wcnt[w];
                idx = (int64_t)p.blockcnt[(int64_t)(c0 + ci) * gridDim.x + blockIdx.x] + before +
                      __popc(bal & ((1u << lane) - 1u));
                if (!vis || idx >= p.cap) continue;
                p.camera_ids[idx] = c0 + ci;
                p.gaussian_ids[idx] = (int32_t)n;
            }
            float4* rec = reinterpret_cast<float4*>(p.splats + idx * GS_SPLAT_FLOATS);
            int2* rad = reinterpret_cast<int2*>(p.radii) + idx;
            if (!vis) {
                *rad = make_int2(0, 0);
                const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                rec[0] = z4;
                rec[1] = z4;
                rec[2] = z4;
                continue;
            }
            // F9/F10: conic and the A.4 compensation (values path, fp32)
            const float cA = c / det, cB = -b / det, cC = a / det;
            float comp = 1.f;
            if (p.antialiased) {
                float det_raw = Sp00 * Sp11 - Sp01 * Sp01;
                comp = sqrtf(fmaxf(0.f, det_raw / det));
            }
            // F14: colour
            float r, g, bl;
            if (DEG < 0) {   // direct RGB; NULL colors (N-D feature mode): the rgb slots are 0
                r = p.colors ? p.colors[3 * n + 0] : 0.f;
                g = p.colors ? p.colors[3 * n + 1] : 0.f;
                bl = p.colors ? p.colors[3 * n + 2] : 0.f;
            } else {
                float ex = mu0 - cc.campos[0], ey = mu1 - cc.campos[1], ez = mu2 - cc.campos[2];
                float en = sqrtf((ex * ex + ey * ey) + ez * ez);
                float Y[NB];
                sh_eval_basis<(DEG < 0 ? 0 : DEG)>(ex / en, ey / en, ez / en, Y);
                // coefficients streamed (16-byte loads; the row stays in L1/L2 for the next
                // camera) instead of held in registers: keeps occupancy up in this HBM-bound kernel
                float acc[3] = {0.5f, 0.5f, 0.5f};
                const float* src = p.colors + n * (int64_t)p.K * 3;
                if (p.vec_colors && (NB * 3) % 4 == 0) {
#pragma unroll
                    for (int i = 0; i < NB * 3 / 4; i++) {
                        const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
                        acc[(4 * i + 0) % 3] += Y[(4 * i + 0) / 3] * v.x;
                        acc[(4 * i + 1) % 3] += Y[(4 * i + 1) / 3] * v.y;
                        acc[(4 * i + 2) % 3] += Y[(4 * i + 2) / 3] * v.z;
                        acc[(4 * i + 3) % 3] += Y[(4 * i + 3) / 3] * v.w;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < NB * 3; i++) acc[i % 3] += Y[i / 3] * __ldg(src + i);
                }
                const float acc0 = acc[0], acc1 = acc[1], acc2 = acc[2];
                r = fmaxf(acc0, 0.f);
                g = fmaxf(acc1, 0.f);
                bl = fmaxf(acc2, 0.f);
            }
            *rad = make_int2(rx, ry);
            rec[0] = make_float4(mx, my, op * comp, tz);
            rec[1] = make_float4(cA, cB, cC, a);      // a = Sigma'_b,xx (support box of K6/K7)
            rec[2] = make_float4(r, g, bl, c);        // c = Sigma'_b,yy
        }
    }
}

}  // namespace

namespace {

// Exclusive scan (in place) of the C * nblk per-(camera, block) counts, camera-major;
// *nnz = total, *overflow = total > cap.  One block, 16 consecutive entries per thread per
// round of 16384.
constexpr int kScanT = 1024, kScanItems = 16;
__global__ void __launch_bounds__(kScanT) k_pack_scan(int* cnt, int64_t n, int64_t cap, int64_t* nnz,
                                                      int32_t* overflow) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_w[kScanT / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t carry = 0;
    for (int64_t r = 0; r < n; r += (int64_t)kScanT * kScanItems) {
        const int64_t i0 = r + (int64_t)threadIdx.x * kScanItems;
        int v[kScanItems];
        int sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            v[k] = i0 + k < n ? cnt[i0 + k] : 0;
            sum += v[k];
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            const int w = s_w[lane];
            int wx = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wx, o);
                if (lane >= o) wx += y;
            }
            s_w[lane] = wx - w;
            if (lane == 31) s_w[32] = wx;
        }
        __syncthreads();
        int64_t run = carry + (x - sum) + s_w[warp];
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            if (i0 + k < n) cnt[i0 + k] = (int)min(run, cap);   // positions >= cap are dropped (overflow)
            run += v[k];
        }
        carry += s_w[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *nnz = carry;
        *overflow = carry > cap ? 1 : 0;
    }
}

ProjParams make_proj_params(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                            const float* quats, const float* scales, const float* opac, const float* colors, int K,
                            const float* viewmats, const float* Ks, int32_t* radii, float* splats) {
    ProjParams p{};
    p.N = N; p.C = C; p.W = W; p.H = H; p.K = K;
    p.near_plane = o.near_plane; p.far_plane = o.far_plane; p.eps2d = o.eps2d; p.alpha_min = o.alpha_min;
    p.antialiased = o.antialiased; p.bbox_mode = o.bbox_mode; p.fov_clamp = o.fov_clamp;
    p.means = means; p.quats = quats; p.scales = scales; p.opac = opac; p.colors = colors;
    p.viewmats = viewmats; p.Ks = Ks; p.radii = radii; p.splats = splats;
    p.vec_colors = ((reinterpret_cast<uintptr_t>(colors) & 15u) == 0) && ((K * 3) % 4 == 0);
    return p;
}

template <int MODE>
void launch_mode(int deg, int grid, const ProjParams& p, cudaStream_t s) {
    switch (deg) {
        case -1: launch_pdl(k_project_fwd<-1, MODE>, dim3(grid), dim3(kThreads), s, p); break;
        case 0: launch_pdl(k_project_fwd<0, MODE>, dim3(grid), dim3(kThreads), s, p); break;
        case 1: launch_pdl(k_project_fwd<1, MODE>, dim3(grid), dim3(kThreads), s, p); break;
        case 2: launch_pdl(k_project_fwd<2, MODE>, dim3(grid), dim3(kThreads), s, p); break;
        default: launch_pdl(k_project_fwd<3, MODE>, dim3(grid), dim3(kThreads), s, p); break;
    }
}

}  // namespace

gs_status launch_project_fwd(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                             const float* quats, const float* scales, const float* opac,
                             const float* colors, int K, const float* viewmats, const float* Ks,
                             int32_t* radii, float* splats, cudaStream_t s) {
    if (N == 0) return GS_OK;
    const ProjParams p = make_proj_params(o, N, C, W, H, means, quats, scales, opac, colors, K, viewmats, Ks, radii,
                                          splats);
    launch_mode<kDense>(o.sh_degree, div_up(N, kThreads), p, s);
    GS_LAUNCH_CHECK("k_project_fwd");
    return GS_OK;
}

size_t project_packed_workspace_bytes(int64_t N, int C) {
    return ((size_t)C * (size_t)div_up(N > 0 ? N : 1, kThreads) * sizeof(int) + 255) & ~(size_t)255;
}

gs_status launch_project_packed(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                                const float* quats, const float* scales, const float* opac, const float* colors,
                                int K, const float* viewmats, const float* Ks, int64_t cap, int64_t* nnz,
                                int32_t* overflow, int32_t* camera_ids, int32_t* gaussian_ids, int32_t* radii,
                                float* splats, void* ws, cudaStream_t s) {
    ProjParams p = make_proj_params(o, N, C, W, H, means, quats, scales, opac, colors, K, viewmats, Ks, radii,
                                    splats);
    const int grid = div_up(N > 0 ? N : 1, kThreads);
    p.blockcnt = static_cast<int*>(ws);
    p.cap = cap;
    p.camera_ids = camera_ids;
    p.gaussian_ids = gaussian_ids;
    if (N > 0) launch_mode<kCount>(o.sh_degree, grid, p, s);
    launch_pdl(k_pack_scan, dim3(1), dim3(kScanT), s, p.blockcnt, N > 0 ? (int64_t)C * grid : 0, cap, nnz, overflow);
    if (N > 0) launch_mode<kPacked>(o.sh_degree, grid, p, s);
    GS_LAUNCH_CHECK("k_project_fwd<packed>");
    return GS_OK;
}

}  // namespace gsb
