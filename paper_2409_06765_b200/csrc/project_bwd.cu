// K8: projection backward -- P1..P9 of SURVEY Appendix A, restating App. C.3-C.4
// of arXiv 2409.06765, with the readings Q10 (mu' -> t re-derived from the
// pinhole map P:790), Q11 (dL/dT symmetric form), Q27 (exact derivative of the clamped J)
// and the A.4 compensation gradient (P3, derived from P:281).
//
// Design (B200): one thread per Gaussian; the thread recomputes the forward quantities
// in registers, loops over the C cameras of the call and sums their contributions
// (no atomics: deterministic, Q30), then writes every parameter gradient once
// (44 B + 12K B per Gaussian, vector stores for SH).  HBM-bound (DESIGN.md roofline K8).
#include "gs_internal.cuh"
#include "sh.cuh"

namespace gsb {
namespace {

constexpr int kThreads = 128;
#ifndef GS_PBWD_MINB
#define GS_PBWD_MINB 5   // 96 registers: 5 CTAs/SM (measured best of 4, 5, 6)
#endif

struct PBParams {
    int64_t N;
    int64_t n_begin, n_end;   // the Gaussians [n_begin, n_end) of this launch; outputs row n - n_begin
    int C, W, H, K;
    float eps2d;
    int antialiased, fov_clamp;
    int vec_colors;   // colors and v_colors bases 16B-aligned and K*3 % 4 == 0
    const float* means;
    const float* quats;
    const float* scales;
    const float* opac;
    const float* colors;
    const float* viewmats;
    const float* Ks;
    const int32_t* radii;
    const float* v_splats;
    const int32_t* map;   // packed mode: (c,n) -> packed item or -1 (else NULL: item = c*N+n)
    float* pose_part;     // pose gradients: per-(block, camera) partial dL/dviewmat rows 0..2 [nblk][C][12]
    float* v_means;
    float* v_quats;
    float* v_scales;
    float* v_opac;
    float* v_colors;
};

// MUFU approximations (relative error ~2^-22): K8 computes values, not decisions, and its
// tolerance is 1e-3 relative (the Q27 clamp branch keeps IEEE divisions)
__device__ __forceinline__ float rcp_fast(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_fast(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// R(q / |q|)
__device__ __forceinline__ void quat_rot(float4 q4, float (&R)[3][3]) {
    const float iq = rsqrt_fast(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
    const float qw = q4.x * iq, qx = q4.y * iq, qy = q4.z * iq, qz = q4.w * iq;
    R[0][0] = 1.f - 2.f * (qy * qy + qz * qz); R[0][1] = 2.f * (qx * qy - qw * qz); R[0][2] = 2.f * (qx * qz + qw * qy);
    R[1][0] = 2.f * (qx * qy + qw * qz); R[1][1] = 1.f - 2.f * (qx * qx + qz * qz); R[1][2] = 2.f * (qy * qz - qw * qx);
    R[2][0] = 2.f * (qx * qz - qw * qy); R[2][1] = 2.f * (qy * qz + qw * qx); R[2][2] = 1.f - 2.f * (qx * qx + qy * qy);
}

// Transposed warp reduction of 16 values: lane l ends with the warp sum of value (l >> 1) & 15.
__device__ __forceinline__ float reduce_scatter16(const float (&v)[16], int lane) {
    float u[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const bool h = lane & 16;
        u[i] = (h ? v[i + 8] : v[i]) + __shfl_xor_sync(0xffffffffu, h ? v[i] : v[i + 8], 16);
    }
    float w[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const bool h = lane & 8;
        w[i] = (h ? u[i + 4] : u[i]) + __shfl_xor_sync(0xffffffffu, h ? u[i] : u[i + 4], 8);
    }
    float x[2];
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const bool h = lane & 4;
        x[i] = (h ? w[i + 2] : w[i]) + __shfl_xor_sync(0xffffffffu, h ? w[i] : w[i + 2], 4);
    }
    const bool h = lane & 2;
    float y = (h ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, h ? x[0] : x[1], 2);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    return y;
}

// POSE: also the camera pose gradients dL/dviewmat (App. pose optimisation, P:233-239,
// P:713-726): per camera, every thread's contribution is reduced over the block and written
// as one per-(block, camera) partial; k_pose_reduce sums the partials in a fixed order.
template <int DEG, bool POSE>
__global__ void __launch_bounds__(kThreads, GS_PBWD_MINB) k_project_bwd(PBParams p) {
    pdl_trigger();
    pdl_wait();
    const int64_t n0 = p.n_begin + (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const bool active = n0 < p.n_end;
    if (!POSE && !active) return;   // without POSE there is no block-level synchronisation below
    const int64_t n = active ? n0 : p.n_end - 1;   // POSE: idle threads read a valid row, contribute nothing
    const int64_t no = n - p.n_begin;              // output row (a chunk's outputs start at n_begin)
    constexpr int NB = DEG < 0 ? 1 : (DEG + 1) * (DEG + 1);
    __shared__ float s_pose[POSE ? kThreads / 32 : 1][12];

    const float mu[3] = {p.means[3 * n], p.means[3 * n + 1], p.means[3 * n + 2]};
    const float4 q4 = reinterpret_cast<const float4*>(p.quats)[n];
    const float s[3] = {p.scales[3 * n], p.scales[3 * n + 1], p.scales[3 * n + 2]};
    const float op = p.opac[n];
    // Sigma = M M^T with M = R(q_hat) S (only Sigma stays live through the camera loop; R and M
    // are recomputed after it -- fewer registers, more warps in flight for this HBM-bound kernel)
    float Sig[3][3];
    {
        float R[3][3], M[3][3];
        quat_rot(q4, R);
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) M[i][j] = R[i][j] * s[j];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) Sig[i][j] = M[i][0] * M[j][0] + M[i][1] * M[j][1] + M[i][2] * M[j][2];
    }

    float g_mu[3] = {0.f, 0.f, 0.f}, g_S[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
    float g_op = 0.f;
    // SH gradient accumulators live in shared memory (one column per thread, conflict-free)
    // and the coefficients are streamed from L1/L2, keeping registers and occupancy for this
    // HBM-bound kernel
    __shared__ float s_gc[DEG < 0 ? 1 : NB * 3][kThreads + 1];   // +1: conflict-free transposed reads
    float g_rgb[3] = {0.f, 0.f, 0.f};
    if (DEG >= 0) {
#pragma unroll
        for (int i = 0; i < NB * 3; i++) s_gc[i][threadIdx.x] = 0.f;
    }
    const float* src = p.colors + n * (int64_t)p.K * 3;
    const bool vec = p.vec_colors && (NB * 3) % 4 == 0;
    bool seen = false;

    for (int c = 0; c < p.C; c++) {
        int64_t idx = (int64_t)c * p.N + n;
        bool vis = active;
        if (vis && p.map) {
            const int m = p.map[idx];
            vis = m >= 0;
            idx = vis ? m : 0;
        }
        if (vis) {
            const int2 rad = reinterpret_cast<const int2*>(p.radii)[idx];
            vis = rad.x > 0 && rad.y > 0;
        }
        float pw[12];   // this thread's dL/dviewmat rows 0..2 for camera c
#pragma unroll
        for (int i = 0; i < 12; i++) pw[i] = 0.f;
        if (vis) {
#ifndef GS_PBWD_PREFETCH
#define GS_PBWD_PREFETCH 1
#endif
            if (GS_PBWD_PREFETCH && DEG > 0 && !seen) {
                // the SH row (12K floats) is needed only after the geometry chain below: start
                // bringing its cache lines into L2 now, so its loads overlap that arithmetic
                const char* row = reinterpret_cast<const char*>(src);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 96));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(row + NB * 12 - 4));
            }
            seen = true;
            const float4* vr = reinterpret_cast<const float4*>(p.v_splats + idx * GS_SPLAT_FLOATS);
            const float4 v0 = vr[0], v1 = vr[1], v2 = vr[2];
            const float* vm = p.viewmats + 16 * (int64_t)c;
            const float* Kc = p.Ks + 9 * (int64_t)c;
            float Wr[3][3], w[3];
#pragma unroll
            for (int i = 0; i < 3; i++) {
#pragma unroll
                for (int j = 0; j < 3; j++) Wr[i][j] = vm[4 * i + j];
                w[i] = vm[4 * i + 3];
            }
            const float fx = Kc[0], fy = Kc[4], cx = Kc[2], cy = Kc[5];
            float t[3];
#pragma unroll
            for (int i = 0; i < 3; i++) t[i] = Wr[i][0] * mu[0] + Wr[i][1] * mu[1] + Wr[i][2] * mu[2] + w[i];
            const float tz = t[2];
            // Sigma_c = Wr Sigma Wr^T
            float A[3][3], Sc[3][3];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) A[i][j] = Wr[i][0] * Sig[0][j] + Wr[i][1] * Sig[1][j] + Wr[i][2] * Sig[2][j];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) Sc[i][j] = A[i][0] * Wr[j][0] + A[i][1] * Wr[j][1] + A[i][2] * Wr[j][2];
            // J with clamp (Q27)
            float txc = t[0], tyc = t[1];
            bool clx = false, cly = false;
            if (p.fov_clamp) {
                const float Wf = (float)p.W, Hf = (float)p.H;
                const float tanx = 0.5f * Wf / fx, tany = 0.5f * Hf / fy;
                const float lxp = (Wf - cx) / fx + 0.3f * tanx, lxn = cx / fx + 0.3f * tanx;
                const float lyp = (Hf - cy) / fy + 0.3f * tany, lyn = cy / fy + 0.3f * tany;
                const float u = t[0] / tz, v = t[1] / tz;
                clx = (u > lxp) || (u < -lxn);
                cly = (v > lyp) || (v < -lyn);
                txc = tz * fminf(lxp, fmaxf(-lxn, u));
                tyc = tz * fminf(lyp, fmaxf(-lyn, v));
            }
            const float rz = rcp_fast(tz), rz2 = rz * rz, rz3 = rz2 * rz;
            const float J[2][3] = {{fx * rz, 0.f, -fx * txc * rz2}, {0.f, fy * rz, -fy * tyc * rz2}};
            float B[2][3], Sp[2][2];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) B[i][j] = J[i][0] * Sc[0][j] + J[i][1] * Sc[1][j] + J[i][2] * Sc[2][j];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 2; j++) Sp[i][j] = B[i][0] * J[j][0] + B[i][1] * J[j][1] + B[i][2] * J[j][2];
            const float a = Sp[0][0] + p.eps2d, b = Sp[0][1], cc = Sp[1][1] + p.eps2d;
            const float detb = a * cc - b * b;
            const float idet = rcp_fast(detb);
            const float Y00 = cc * idet, Y01 = -b * idet, Y11 = a * idet;
            float comp = 1.f, det_raw = 0.f;
            if (p.antialiased) {
                det_raw = Sp[0][0] * Sp[1][1] - Sp[0][1] * Sp[0][1];
                comp = sqrtf(fmaxf(0.f, det_raw * idet));
            }
            // ---- P1: o_eff = o * comp
            const float v_oeff = v0.z;
            g_op += v_oeff * comp;
            const float v_comp = v_oeff * op;
            // ---- P2: v_Spb = -Y G_Y Y, G_Y = [[vA, vB/2],[vB/2, vC]]
            const float gA = v0.w, gB = 0.5f * v1.x, gC = v1.y;   // gradient slots 3-5 (include/gs.h)
            const float YG00 = Y00 * gA + Y01 * gB, YG01 = Y00 * gB + Y01 * gC;
            const float YG10 = Y01 * gA + Y11 * gB, YG11 = Y01 * gB + Y11 * gC;
            float vS00 = -(YG00 * Y00 + YG01 * Y01);
            float vS01 = -(YG00 * Y01 + YG01 * Y11);
            float vS11 = -(YG10 * Y01 + YG11 * Y11);
            // ---- P3 (AA): + v_comp * comp/2 * (Sigma'^-1 - Spb^-1)
            if (p.antialiased && det_raw > 0.f) {
                const float k = v_comp * 0.5f * comp;
                const float idr = rcp_fast(det_raw);
                vS00 += k * (Sp[1][1] * idr - Y00);
                vS01 += k * (-Sp[0][1] * idr - Y01);
                vS11 += k * (Sp[0][0] * idr - Y11);
            }
            const float vSp[2][2] = {{vS00, vS01}, {vS01, vS11}};
            // ---- P4: v_Sc = J^T vSp J; v_J = 2 vSp J Sc (Q11)
            float vSc[3][3], vJ[2][3];
            float PJ[2][3];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) PJ[i][j] = vSp[i][0] * J[0][j] + vSp[i][1] * J[1][j];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) vSc[i][j] = J[0][i] * PJ[0][j] + J[1][i] * PJ[1][j];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) vJ[i][j] = 2.f * (PJ[i][0] * Sc[0][j] + PJ[i][1] * Sc[1][j] + PJ[i][2] * Sc[2][j]);
            // ---- P5: v_t through J (exact with clamp Q27) and mu' (Q10)
            float vt0 = 0.f, vt1 = 0.f, vt2 = -fx * rz2 * vJ[0][0] - fy * rz2 * vJ[1][1];
            if (!clx) {
                vt0 += -fx * rz2 * vJ[0][2];
                vt2 += 2.f * fx * t[0] * rz3 * vJ[0][2];
            } else {
                vt2 += fx * txc * rz3 * vJ[0][2];
            }
            if (!cly) {
                vt1 += -fy * rz2 * vJ[1][2];
                vt2 += 2.f * fy * t[1] * rz3 * vJ[1][2];
            } else {
                vt2 += fy * tyc * rz3 * vJ[1][2];
            }
            vt0 += fx * rz * v0.x;
            vt1 += fy * rz * v0.y;
            vt2 -= fx * t[0] * rz2 * v0.x + fy * t[1] * rz2 * v0.y;
            vt2 += v2.y;   // depth = t_z (F4), the depth-rendering gradient (slot 9)
            if constexpr (POSE) {
                // t = W mu + w: dL/dW += v_t mu^T, dL/dw += v_t
                const float vt[3] = {vt0, vt1, vt2};
#pragma unroll
                for (int i = 0; i < 3; i++) {
#pragma unroll
                    for (int j = 0; j < 3; j++) pw[4 * i + j] += vt[i] * mu[j];
                    pw[4 * i + 3] += vt[i];
                }
            }
            if constexpr (POSE) {
                // Sigma_c = W Sigma W^T (Fig. P:423): dL/dW += (vSc + vSc^T) W Sigma, W Sigma = A
#pragma unroll
                for (int i = 0; i < 3; i++)
#pragma unroll
                    for (int j = 0; j < 3; j++)
                        pw[4 * i + j] += (vSc[i][0] + vSc[0][i]) * A[0][j] + (vSc[i][1] + vSc[1][i]) * A[1][j] +
                                         (vSc[i][2] + vSc[2][i]) * A[2][j];
            }
            // ---- P6: v_mu += W^T v_t; v_Sigma += W^T v_Sc W
#pragma unroll
            for (int i = 0; i < 3; i++) g_mu[i] += Wr[0][i] * vt0 + Wr[1][i] * vt1 + Wr[2][i] * vt2;
            float T1[3][3];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) T1[i][j] = vSc[i][0] * Wr[0][j] + vSc[i][1] * Wr[1][j] + vSc[i][2] * Wr[2][j];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) g_S[i][j] += Wr[0][i] * T1[0][j] + Wr[1][i] * T1[1][j] + Wr[2][i] * T1[2][j];
            // ---- P7: colour
            if (DEG < 0) {
                g_rgb[0] += v1.z;   // gradient slots 6-8
                g_rgb[1] += v1.w;
                g_rgb[2] += v2.x;
            } else {
                float campos[3];
#pragma unroll
                for (int i = 0; i < 3; i++) campos[i] = -(Wr[0][i] * w[0] + Wr[1][i] * w[1] + Wr[2][i] * w[2]);
                const float ex = mu[0] - campos[0], ey = mu[1] - campos[1], ez = mu[2] - campos[2];
                const float ren = rsqrt_fast(ex * ex + ey * ey + ez * ez);
                const float dx = ex * ren, dy = ey * ren, dz = ez * ren;
                float Yb[NB];
                sh_eval_basis<(DEG < 0 ? 0 : DEG)>(dx, dy, dz, Yb);
                float raw[3] = {0.5f, 0.5f, 0.5f};
                if (vec) {
#pragma unroll
                    for (int i = 0; i < NB * 3 / 4; i++) {
                        const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
                        raw[(4 * i + 0) % 3] += Yb[(4 * i + 0) / 3] * v.x;
                        raw[(4 * i + 1) % 3] += Yb[(4 * i + 1) / 3] * v.y;
                        raw[(4 * i + 2) % 3] += Yb[(4 * i + 2) / 3] * v.z;
                        raw[(4 * i + 3) % 3] += Yb[(4 * i + 3) / 3] * v.w;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < NB * 3; i++) raw[i % 3] += Yb[i / 3] * __ldg(src + i);
                }
                const float vr[3] = {raw[0] > 0.f ? v1.z : 0.f, raw[1] > 0.f ? v1.w : 0.f, raw[2] > 0.f ? v2.x : 0.f};
#pragma unroll
                for (int i = 0; i < NB * 3; i++) s_gc[i][threadIdx.x] += Yb[i / 3] * vr[i % 3];
                if (DEG > 0) {
                    float wj[NB];
#pragma unroll
                    for (int j = 0; j < NB; j++) wj[j] = 0.f;
                    if (vec) {
#pragma unroll
                        for (int i = 0; i < NB * 3 / 4; i++) {
                            const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
                            wj[(4 * i + 0) / 3] += v.x * vr[(4 * i + 0) % 3];
                            wj[(4 * i + 1) / 3] += v.y * vr[(4 * i + 1) % 3];
                            wj[(4 * i + 2) / 3] += v.z * vr[(4 * i + 2) % 3];
                            wj[(4 * i + 3) / 3] += v.w * vr[(4 * i + 3) % 3];
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < NB * 3; i++) wj[i / 3] += __ldg(src + i) * vr[i % 3];
                    }
                    float gx = 0.f, gy = 0.f, gz = 0.f;
                    sh_basis_vjp<(DEG < 0 ? 0 : DEG)>(dx, dy, dz, wj, gx, gy, gz);
                    const float dd = dx * gx + dy * gy + dz * gz;
                    const float ve[3] = {(gx - dx * dd) * ren, (gy - dy * dd) * ren, (gz - dz * dd) * ren};
                    g_mu[0] += ve[0];
                    g_mu[1] += ve[1];
                    g_mu[2] += ve[2];
                    if constexpr (POSE) {
                        // e = mu - campos, campos = -W^T w: dL/dW_ki += ve_i w_k, dL/dw_k += (W ve)_k
#pragma unroll
                        for (int k = 0; k < 3; k++) {
#pragma unroll
                            for (int i = 0; i < 3; i++) pw[4 * k + i] += ve[i] * w[k];
                            pw[4 * k + 3] += Wr[k][0] * ve[0] + Wr[k][1] * ve[1] + Wr[k][2] * ve[2];
                        }
                    }
                }
            }
            (void)cy;
            (void)cx;
        }  // vis
        if constexpr (POSE) {
            float v16[16];
#pragma unroll
            for (int i = 0; i < 16; i++) v16[i] = i < 12 ? pw[i] : 0.f;
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            const float r = reduce_scatter16(v16, lane);
            if ((lane & 1) == 0 && (lane >> 1) < 12) s_pose[warp][lane >> 1] = r;
            __syncthreads();
            if (threadIdx.x < 12) {
                float t = 0.f;
#pragma unroll
                for (int w2 = 0; w2 < kThreads / 32; w2++) t += s_pose[w2][threadIdx.x];
                p.pose_part[((int64_t)blockIdx.x * p.C + c) * 12 + threadIdx.x] = t;
            }
            __syncthreads();
        }
    }
    if (!active) return;

    // ---- P8: v_M = (vS + vS^T) M; v_s_j = (R^T v_M)_jj; v_R = v_M S
    const float rq = rsqrt_fast(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
    const float qw = q4.x * rq, qx = q4.y * rq, qy = q4.z * rq, qz = q4.w * rq;
    float R[3][3], M[3][3];
    quat_rot(q4, R);
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) M[i][j] = R[i][j] * s[j];
    float vM[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            vM[i][j] = (g_S[i][0] + g_S[0][i]) * M[0][j] + (g_S[i][1] + g_S[1][i]) * M[1][j] +
                       (g_S[i][2] + g_S[2][i]) * M[2][j];
    float gsc[3];
#pragma unroll
    for (int j = 0; j < 3; j++) gsc[j] = R[0][j] * vM[0][j] + R[1][j] * vM[1][j] + R[2][j] * vM[2][j];
    float vR[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) vR[i][j] = vM[i][j] * s[j];
    // ---- P9: dR/d(w,x,y,z) at q_hat, then the normalisation
    const float w_ = qw, x_ = qx, y_ = qy, z_ = qz;
    float vqw = 2.f * (-z_ * vR[0][1] + y_ * vR[0][2] + z_ * vR[1][0] - x_ * vR[1][2] - y_ * vR[2][0] + x_ * vR[2][1]);
    float vqx = 2.f * (y_ * vR[0][1] + z_ * vR[0][2] + y_ * vR[1][0] - 2.f * x_ * vR[1][1] - w_ * vR[1][2] +
                       z_ * vR[2][0] + w_ * vR[2][1] - 2.f * x_ * vR[2][2]);
    float vqy = 2.f * (-2.f * y_ * vR[0][0] + x_ * vR[0][1] + w_ * vR[0][2] + x_ * vR[1][0] + z_ * vR[1][2] -
                       w_ * vR[2][0] + z_ * vR[2][1] - 2.f * y_ * vR[2][2]);
    float vqz = 2.f * (-2.f * z_ * vR[0][0] - w_ * vR[0][1] + x_ * vR[0][2] + w_ * vR[1][0] - 2.f * z_ * vR[1][1] +
                       y_ * vR[1][2] + x_ * vR[2][0] + y_ * vR[2][1]);
    const float dot = vqw * w_ + vqx * x_ + vqy * y_ + vqz * z_;
    float4 oq = make_float4((vqw - dot * w_) * rq, (vqx - dot * x_) * rq, (vqy - dot * y_) * rq, (vqz - dot * z_) * rq);
    if (!seen) {   // culled in every camera (includes zero / non-finite quaternions): zeros
        oq = make_float4(0.f, 0.f, 0.f, 0.f);
        gsc[0] = gsc[1] = gsc[2] = 0.f;
    }
    reinterpret_cast<float4*>(p.v_quats)[no] = oq;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        p.v_means[3 * no + i] = g_mu[i];
        p.v_scales[3 * no + i] = gsc[i];
    }
    p.v_opac[no] = g_op;
    if (DEG < 0) {
        if (p.v_colors) {   // NULL in N-D feature mode: the raster backward wrote the feature gradient
#pragma unroll
            for (int i = 0; i < 3; i++) p.v_colors[3 * no + i] = g_rgb[i];
        }
    } else {
        const int lane = threadIdx.x & 31, wslot = threadIdx.x & ~31;
        const int64_t wbase = no - lane;
        constexpr int F = NB * 3;   // floats per Gaussian
        if (vec && p.K == NB && wbase + 32 <= p.n_end - p.n_begin) {
            // the warp's 32 consecutive rows are one contiguous block: transpose through shared
            // memory and write it with coalesced 16-byte stores
            __syncwarp();
            float4* dstw = reinterpret_cast<float4*>(p.v_colors + wbase * F);
#pragma unroll 4
            for (int c = lane; c < 32 * F / 4; c += 32) {
                float v[4];
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int f = 4 * c + e;
                    v[e] = s_gc[f % F][wslot + f / F];
                }
                dstw[c] = make_float4(v[0], v[1], v[2], v[3]);
            }
        } else {
            float* dst = p.v_colors + no * (int64_t)p.K * 3;
#pragma unroll
            for (int i = 0; i < NB * 3; i++) dst[i] = s_gc[i][threadIdx.x];
            for (int i = NB * 3; i < p.K * 3; i++) dst[i] = 0.f;
        }
    }
}

}  // namespace

namespace {

PBParams make_pb_params(const gs_options& o, int64_t N, int C, int W, int H, const float* means, const float* quats,
                        const float* scales, const float* opac, const float* colors, int K, const float* viewmats,
                        const float* Ks, const int32_t* radii, const float* v_splats, float* v_means,
                        float* v_quats, float* v_scales, float* v_opac, float* v_colors) {
    PBParams p{};
    p.N = N; p.C = C; p.W = W; p.H = H; p.K = K;
    p.n_begin = 0; p.n_end = N;
    p.eps2d = o.eps2d; p.antialiased = o.antialiased; p.fov_clamp = o.fov_clamp;
    p.means = means; p.quats = quats; p.scales = scales; p.opac = opac; p.colors = colors;
    p.viewmats = viewmats; p.Ks = Ks; p.radii = radii; p.v_splats = v_splats; p.map = nullptr;
    // float4 path reads colors and writes v_colors: both bases must be 16-byte aligned
    p.vec_colors = ((reinterpret_cast<uintptr_t>(v_colors) & 15u) == 0) &&
                   ((reinterpret_cast<uintptr_t>(colors) & 15u) == 0) && ((K * 3) % 4 == 0);
    p.v_means = v_means; p.v_quats = v_quats; p.v_scales = v_scales; p.v_opac = v_opac; p.v_colors = v_colors;
    return p;
}

template <bool POSE>
void launch_pb_t(int deg, const PBParams& p, cudaStream_t s) {
    const int grid = div_up(p.n_end - p.n_begin, kThreads);
    switch (deg) {
        case -1: launch_pdl(k_project_bwd<-1, POSE>, dim3(grid), dim3(kThreads), s, p); break;
        case 0: launch_pdl(k_project_bwd<0, POSE>, dim3(grid), dim3(kThreads), s, p); break;
        case 1: launch_pdl(k_project_bwd<1, POSE>, dim3(grid), dim3(kThreads), s, p); break;
        case 2: launch_pdl(k_project_bwd<2, POSE>, dim3(grid), dim3(kThreads), s, p); break;
        default: launch_pdl(k_project_bwd<3, POSE>, dim3(grid), dim3(kThreads), s, p); break;
    }
}

// dL/dviewmat[c] = sum over blocks of the per-(block, camera) partials, in block order
// (deterministic); row 3 of the 4x4 is not a parameter of the projection: 0.
constexpr int kPoseT = 120;   // 12 values x 10 lanes each
__global__ void __launch_bounds__(kPoseT) k_pose_reduce(const float* __restrict__ part, int nblk, int C,
                                                      float* __restrict__ v_viewmats) {
    pdl_trigger();
    pdl_wait();
    __shared__ float s_acc[kPoseT];
    const int c = blockIdx.x, v = threadIdx.x / 10, r = threadIdx.x % 10;
    float t = 0.f;
    for (int b = r; b < nblk; b += 10) t += part[((int64_t)b * C + c) * 12 + v];
    s_acc[threadIdx.x] = t;
    __syncthreads();
    if (r == 0) {
        float u = 0.f;
        for (int k = 0; k < 10; k++) u += s_acc[threadIdx.x + k];
        v_viewmats[16 * (int64_t)c + v] = u;
    }
    if (threadIdx.x < 4) v_viewmats[16 * (int64_t)c + 12 + threadIdx.x] = 0.f;
}

gs_status launch_pb(int deg, PBParams p, float* v_viewmats, void* pose_ws, cudaStream_t s) {
    if (!v_viewmats) {
        launch_pb_t<false>(deg, p, s);
        return GS_OK;
    }
    p.pose_part = static_cast<float*>(pose_ws);
    launch_pb_t<true>(deg, p, s);
    launch_pdl(k_pose_reduce, dim3(p.C), dim3(kPoseT), s, p.pose_part, div_up(p.n_end - p.n_begin, kThreads), p.C,
               v_viewmats);
    return GS_OK;
}

// map[camera_ids[i] * N + gaussian_ids[i]] = i for the live packed items (map pre-set to -1)
__global__ void k_pack_map(const int32_t* __restrict__ cam, const int32_t* __restrict__ gid, const int64_t* d_nnz,
                           int64_t cap, int64_t N, int32_t* __restrict__ map) {
    pdl_trigger();
    pdl_wait();
    const int64_t n = min(*d_nnz, cap);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) map[(int64_t)cam[i] * N + gid[i]] = (int32_t)i;
}

}  // namespace

gs_status launch_project_bwd(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                             const float* quats, const float* scales, const float* opac,
                             const float* colors, int K, const float* viewmats, const float* Ks,
                             const int32_t* radii, const float* v_splats, float* v_means,
                             float* v_quats, float* v_scales, float* v_opac, float* v_colors,
                             float* v_viewmats, void* ws, cudaStream_t s) {
    if (N == 0) {
        if (v_viewmats && cudaMemsetAsync(v_viewmats, 0, sizeof(float) * 16 * (size_t)C, s) != cudaSuccess)
            return GS_ERR_CUDA;
        return GS_OK;
    }
    const PBParams p = make_pb_params(o, N, C, W, H, means, quats, scales, opac, colors, K, viewmats, Ks, radii,
                                      v_splats, v_means, v_quats, v_scales, v_opac, v_colors);
    launch_pb(o.sh_degree, p, v_viewmats, ws, s);
    GS_LAUNCH_CHECK("k_project_bwd");
    return GS_OK;
}

gs_status launch_project_bwd_range(const gs_options& o, int64_t N, int64_t n_begin, int64_t n_end, int C, int W,
                                   int H, const float* means, const float* quats, const float* scales,
                                   const float* opac, const float* colors, int K, const float* viewmats,
                                   const float* Ks, const int32_t* radii, const float* v_splats, float* v_means,
                                   float* v_quats, float* v_scales, float* v_opac, float* v_colors, cudaStream_t s) {
    if (n_end <= n_begin) return GS_OK;
    PBParams p = make_pb_params(o, N, C, W, H, means, quats, scales, opac, colors, K, viewmats, Ks, radii, v_splats,
                                v_means, v_quats, v_scales, v_opac, v_colors);
    p.n_begin = n_begin;
    p.n_end = n_end;
    launch_pb(o.sh_degree, p, nullptr, nullptr, s);
    GS_LAUNCH_CHECK("k_project_bwd<range>");
    return GS_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t project_bwd_workspace_bytes(int64_t N, int C) {
    return align256((size_t)div_up(N > 0 ? N : 1, kThreads) * (size_t)C * 12 * sizeof(float));
}

size_t project_bwd_packed_workspace_bytes(int64_t N, int C) {
    return align256((size_t)C * (size_t)N * sizeof(int32_t)) + project_bwd_workspace_bytes(N, C);
}

gs_status launch_project_bwd_packed(const gs_options& o, int64_t N, int C, int W, int H, const float* means,
                                    const float* quats, const float* scales, const float* opac,
                                    const float* colors, int K, const float* viewmats, const float* Ks,
                                    int64_t cap, const int64_t* nnz, const int32_t* camera_ids,
                                    const int32_t* gaussian_ids, const int32_t* radii, const float* v_splats,
                                    float* v_means, float* v_quats, float* v_scales, float* v_opac,
                                    float* v_colors, float* v_viewmats, void* ws, cudaStream_t s) {
    if (N == 0) {
        if (v_viewmats && cudaMemsetAsync(v_viewmats, 0, sizeof(float) * 16 * (size_t)C, s) != cudaSuccess)
            return GS_ERR_CUDA;
        return GS_OK;
    }
    int32_t* map = static_cast<int32_t*>(ws);
    void* pose_ws = static_cast<char*>(ws) + align256((size_t)C * (size_t)N * sizeof(int32_t));
    if (cudaMemsetAsync(map, 0xff, sizeof(int32_t) * (size_t)C * (size_t)N, s) != cudaSuccess) {
        GS_LAUNCH_CHECK("packed map memset");
        return GS_ERR_CUDA;
    }
    if (cap > 0) launch_pdl(k_pack_map, dim3(div_up(cap, 256)), dim3(256), s, camera_ids, gaussian_ids, nnz, cap, N, map);
    PBParams p = make_pb_params(o, N, C, W, H, means, quats, scales, opac, colors, K, viewmats, Ks, radii, v_splats,
                                v_means, v_quats, v_scales, v_opac, v_colors);
    p.map = map;
    launch_pb(o.sh_degree, p, v_viewmats, pose_ws, s);
    GS_LAUNCH_CHECK("k_project_bwd<packed>");
    return GS_OK;
}

}  // namespace gsb
