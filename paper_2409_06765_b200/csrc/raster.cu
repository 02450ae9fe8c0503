// Stage 3 (K6) and stage 4a (K7): per-pixel compositing forward and backward -- R1..R3 and
// B1..B6 of SURVEY Appendix A, restating App. B.2 and App. C.2 of
// arXiv 2409.06765.
//
// Design (B200).  One CTA per 16x16 tile, one thread per pixel, each warp owning an
// 8x4 pixel block.  The tile's depth-sorted range is walked in batches of 256 splats: each
// batch is gathered from the 48-byte projected records (L2-resident at 1-MP scale) into
// shared memory once and broadcast to all pixels.  While staging, every splat also gets an
// 8-bit mask of the warps whose pixels can see it with alpha >= alpha_min: the
// axis-aligned box of the ellipse sigma <= ln(o/alpha_min), from the blurred variances a, c
// of the record, inflated by a margin that covers fp32 rounding and the ex2/lg2
// approximations.  Each warp then compacts the batch to its own list (ballot, order
// preserving) and walks only that list.  Pixels outside the box would have computed
// alpha < alpha_min and been skipped anyway (Q14), so the result is bit-identical to
// walking every splat; only instruction issue is saved (these kernels are FP32/MUFU issue
// bound, DESIGN.md roofline K6/K7).  The conic is pre-scaled by -log2(e) at staging so the
// per-pair exponent is two FMAs and one MUFU.EX2.  Forward and backward evaluate alpha with
// the same _rn operations (K7 inlines eval_alpha's sequence), so the backward's skip
// decisions replay the forward's bit for bit.  Independent fp32 pairs run as sm_100a packed
// FP32x2 instructions (FADD2 / FMUL2 / FFMA2: one issue slot, identical roundings).  The
// backward reduces each splat's gradient values across the warp with a transposed
// (reduce-scatter) shuffle tree -- 9 shuffles for 8 values instead of 40 -- and lanes holding
// distinct values issue one fp32 reduction each.
#include <type_traits>

#include "gs_internal.cuh"

namespace gsb {
namespace {

constexpr int kThreads = GS_BLOCK_PIXELS; // one thread per pixel of the 16x16 tile
constexpr int kWarps = kThreads / 32;
constexpr int kBatchFwd = 512;            // splats per staged batch: forward (2 per thread) ...
#ifndef GS_K7_BATCH
#define GS_K7_BATCH 256
#endif
constexpr int kBatchBwd = GS_K7_BATCH;            // ... backward (1 per thread; keeps its registers at 48)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16-byte shared-memory load from a 32-bit shared-window address (hoisted base: keeps the
// shared-window base computation out of the inner loops).
__device__ __forceinline__ float4 lds4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// Pre-scaled conic, staged as (a', c', b', b'/2): p = a' dx^2 + c' dy^2 + b' dx dy =
// -sigma * log2(e).  a', c' sit in one aligned register pair so the backward's
// d sigma / d mu' = Sigma'^-1 Delta is one packed multiply and one packed FMA with the b'/2
// lane broadcast (sm_100a FMUL2 / FFMA2, below).
__device__ __forceinline__ float4 prescale_conic(float A, float B, float C) {
    return make_float4(__fmul_rn(-0.5f * kLog2e, A), __fmul_rn(-0.5f * kLog2e, C), __fmul_rn(-kLog2e, B),
                       __fmul_rn(-0.5f * kLog2e, B));
}

// Packed FP32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2): two IEEE round-to-nearest fp32
// operations in one issue slot, each rounded exactly like the scalar _rn operation, with
// scalar operands broadcast and pair halves swapped for free.  K6 / K7 are issue bound (FMA
// pipe ~35 % busy), so pairing independent operations saves issue slots without
// changing a single rounding.
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }

// alpha of one (pixel, splat) pair; returns false when the pair is skipped (sigma < 0 or
// alpha < alpha_min, Q14).  G = exp(-sigma).  Bit-identical in K6 and K7: Delta = mu' - p is
// one packed add of the negated pixel centre npc = (-p.x, -p.y) (x + (-y) == x - y in IEEE),
// the squares one packed multiply.
__device__ __forceinline__ bool eval_alpha(float mx, float my, float o, float4 con, float2 npc, float alpha_max,
                                           float alpha_min, float& dx, float& dy, float& G, float& alpha) {
    const float2 d = add2(make_float2(mx, my), npc);   // Delta = mu' - p (Q21)
    dx = d.x;
    dy = d.y;
    const float2 sq = mul2(d, d);
    const float p = __fmaf_rn(con.z, __fmul_rn(dx, dy), __fmaf_rn(con.x, sq.x, __fmul_rn(con.y, sq.y)));
    if (p > 0.f) return false;   // sigma < 0
    G = ex2_approx(p);
    alpha = fminf(alpha_max, __fmul_rn(o, G));
    return alpha >= alpha_min;
}

// Conservative support of a splat inside its tile.  The set a pixel can take the splat
// from is the ellipse E: sigma(d) = 1/2 (A dx^2 + C dy^2) + B dx dy <= tau, tau =
// ln(o / alpha_min) (alpha = min(alpha_max, o G) < alpha_min outside it, Q14), with
// (A, B, C) the fp32 conic of the record and a, c its blurred variances.  Margins make the
// test conservative with respect to the kernel's fp32 arithmetic: tau is inflated by 0.4 %
// + 4e-3 (lg2.approx, ex2.approx and the rounding of the exponent are all < 1e-5
// relative), every extent by eps = 1e-6 cond (cond = a A = a c / det bounds the relative
// error of the fp32 conic and of the fp32 determinant below) plus 1e-2 px.
//
// Per row r of 4-pixel-high blocks (pixel centres y0 + 4r + 0.5 ... + 3.5) the x-extent of
// E over that slab is [L_r, R_r]: with the exact x-bounds of E at height dy
//   x_+-(dy) = (-B dy +- sqrt(2 A tau - det dy^2)) / A,     det = A C - B^2,
// x_+ is concave and peaks at the rightmost point dy_R = -B hx / C (hx = sqrt(2 tau a)),
// x_- is convex with its minimum at -dy_R, so R_r = x_+(clamp(dy_R, slab)) and
// L_r = x_-(clamp(-dy_R, slab)).  The result is a 4-bit mask of 4-pixel-wide columns per
// row: bit 4 r + k of the returned 16-bit mask is the 4x4 block at column k, row r.
// Ill-conditioned conics (eps >= 1e-2) fall back to the axis-aligned box of E.
// Approximate MUFU square root / reciprocal (relative error ~2^-22): the support test
// below only needs them inside its margins.
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx_f(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t support_mask16(float mx, float my, float o, float A, float B, float Cc, float a,
                                                   float c, float x0, float y0, float alpha_min) {
    if (o < alpha_min * 0.9999f) return 0u;   // alpha = min(alpha_max, o G) <= o (G <= 1)
    float tau = fmaxf(0.f, __logf(__fdividef(o, alpha_min)));
    tau = tau * 1.004f + 4e-3f;
    const float eps = 1e-6f * a * A;
    const float grow = 1.f + eps;
    const float hx0 = sqrt_approx(2.f * tau * a), hy0 = sqrt_approx(2.f * tau * c);
    const float hx = hx0 * grow + 1e-2f;
    const float hy = hy0 * grow + 1e-2f;
    if (!(hx < 1e30f) || !(hy < 1e30f)) return 0xffffu;
    const float u = mx - x0, v = my - y0;
    const bool ell = eps < 1e-2f;
    const float mfrac = 2.f * sqrt_approx(eps) + eps;
    const float mxm = hx0 * mfrac + 1e-2f, mym = hy0 * mfrac + 1e-2f;
    const float det = A * Cc - B * B;
    const float s2 = 2.f * A * tau;
    const float iA = rcp_approx_f(A);
    const float dyR = -B * hx0 * rcp_approx_f(Cc);
    uint32_t m = 0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const float lo = (float)(r * 4) + 0.5f - v, hi = lo + 3.f;   // slab in dy = y - my
        if (!(hi >= -hy && lo <= hy)) continue;
        float L = -hx, R = hx;
        if (ell) {
            const float ylo = lo - mym, yhi = hi + mym;
            const float d1 = fminf(fmaxf(dyR, ylo), yhi);
            const float d2 = fminf(fmaxf(-dyR, ylo), yhi);
            const float R1 = (-B * d1 + sqrt_approx(fmaxf(0.f, s2 - det * d1 * d1))) * iA + mxm;
            const float L1 = (-B * d2 - sqrt_approx(fmaxf(0.f, s2 - det * d2 * d2))) * iA - mxm;
            R = fminf(R, R1);
            L = fmaxf(L, L1);
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float xlo = (float)(k * 4) + 0.5f, xhi = xlo + 3.f;
            if (u + R >= xlo && u + L <= xhi) m |= 1u << (4 * r + k);
        }
    }
    return m;
}

// 8-bit mask of the 8x4 warp blocks (bit 2 r + w for the block at column w, row r): the
// union of the two 4x4 blocks it covers.
__device__ __forceinline__ uint32_t support_mask8(uint32_t m16) {
    uint32_t m = 0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const uint32_t row = (m16 >> (4 * r)) & 0xfu;
        m |= ((row & 3u) ? 1u : 0u) << (2 * r);
        m |= ((row & 12u) ? 1u : 0u) << (2 * r + 1);
    }
    return m;
}

struct RasterParams {
    int C, W, H, TX, TY;
    int64_t N;
    float alpha_max, alpha_min, t_min;
    int cull;                    // 1: conservative alpha-support test per (splat, 4x4 block); 0: every pair
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
    // depth rendering (App. depth rendering): 0 off, 1 accumulated, 2 expected
    int depth_mode;
    float* out_depth;            // fwd output; bwd reads it (expected depth, mode 2)
    const float* v_depth;        // bwd: dL/d out_depth
    // N-D features: 4 channels [c0, c0+4) of feats [n_gauss, D] per pass
    const float* feats;
    int D, c0, first_pass;
    const int32_t* gids;         // packed mode: Gaussian of each record (dense: id - cam N)
    float* out_feats;            // fwd: [C,H,W,D]
    const float* v_feats_img;    // bwd: dL/d out_feats [C,H,W,D]
    float* v_feats;              // bwd: [n_gauss, D] accumulated
    // diagnostics (gs_rasterize_stats)
    int32_t* n_eval;
    int32_t* n_contrib;
    int32_t* n_term;
    // support masks of every staged (intersection) slot, written by K6 and read back by K7
    // (NULL: K7 recomputes them)
    uint16_t* smask;
    // launch order of the (camera, tile) bins (NULL: blockIdx order; gs_tile_order)
    const int32_t* order;
};

// (camera, tile) bin of this CTA
__device__ __forceinline__ void cta_bin(const RasterParams& p, int& tile, int& cam) {
    if (p.order) {
        const int b = p.order[blockIdx.y * gridDim.x + blockIdx.x];
        const int TT = p.TX * p.TY;
        cam = b / TT;
        tile = b - cam * TT;
    } else {
        tile = blockIdx.x;
        cam = blockIdx.y;
    }
}

// Gaussian of a record (dense ids are c*N + n; packed records carry it in gids)
__device__ __forceinline__ int64_t gauss_of(const RasterParams& p, int32_t g, int cam) {
    return p.gids ? (int64_t)p.gids[g] : (int64_t)g - (int64_t)cam * p.N;
}

// Channels [c0, c0 + 4) of a Gaussian's feature row (zeros past D)
__device__ __forceinline__ float4 load_feat4(const RasterParams& p, int32_t g, int cam) {
    const float* f = p.feats + gauss_of(p, g, cam) * p.D + p.c0;
    const int m = p.D - p.c0;
    return make_float4(__ldg(f), m > 1 ? __ldg(f + 1) : 0.f, m > 2 ? __ldg(f + 2) : 0.f, m > 3 ? __ldg(f + 3) : 0.f);
}

struct PixelCoord {
    int px, py, warp, lane;
    bool inside;
    float fpx, fpy, x0, y0;
};

__device__ __forceinline__ PixelCoord pixel_coord(const RasterParams& p, int tile) {
    PixelCoord c;
    c.warp = threadIdx.x >> 5;
    c.lane = threadIdx.x & 31;
    const int tx = tile % p.TX, ty = tile / p.TX;
    c.px = tx * GS_TILE + (c.warp & 1) * 8 + (c.lane & 7);
    c.py = ty * GS_TILE + (c.warp >> 1) * 4 + (c.lane >> 3);
    c.inside = c.px < p.W && c.py < p.H;
    c.fpx = (float)c.px + 0.5f;   // pixel centre
    c.fpy = (float)c.py + 0.5f;
    c.x0 = (float)(tx * GS_TILE);
    c.y0 = (float)(ty * GS_TILE);
    return c;
}

template <int kBatch>
struct Stage {
    float4 xyo[kBatch];   // mean2d.x, mean2d.y, opac_eff, (unused)
    float4 con[kBatch];   // pre-scaled conic
    float4 rgb[kBatch];   // rgb, (unused)
    int32_t id[kBatch];
    uint8_t mask[kBatch];
    // per-warp compacted slot lists (8-bit slots when they fit: fewer registers in K7)
    typename std::conditional<(kBatch <= 256), uint8_t, uint16_t>::type list[kWarps][kBatch];
};

// ID_IN_W: the record id replaces the (unused) depth in the staged xyo.w, so the walk gets it
// with the position load instead of a separate shared-memory access
template <bool FEAT, bool ID_IN_W = false, class StageT>
__device__ __forceinline__ void stage_splat(const RasterParams& p, StageT& s, int slot, int idx, float x0, float y0,
                                            int cam) {
    const int32_t g = p.ids[idx];
    const float4* rec = reinterpret_cast<const float4*>(p.splats + (int64_t)g * GS_SPLAT_FLOATS);
    const float4 r0 = __ldg(rec), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2);
    s.xyo[slot] = ID_IN_W ? make_float4(r0.x, r0.y, r0.z, __int_as_float(g)) : r0;
    s.con[slot] = prescale_conic(r1.x, r1.y, r1.z);
    s.rgb[slot] = FEAT ? load_feat4(p, g, cam) : r2;
    s.id[slot] = g;
    const uint32_t m16 = p.smask ? (uint32_t)p.smask[idx]
                         : (p.cull ? support_mask16(r0.x, r0.y, r0.z, r1.x, r1.y, r1.z, r1.w, r2.w, x0, y0, p.alpha_min)
                                   : 0xffffu);
    s.mask[slot] = (uint8_t)support_mask8(m16);
}

// Order-preserving compaction of the batch slots [0, n) whose mask has this warp's bit
// (and, in the backward, slot index <= max_slot).  Returns the list length.
template <class StageT>
__device__ __forceinline__ int build_warp_list(StageT& s, int n, int warp, int lane, int max_slot) {
    int cnt = 0;
    for (int c = 0; c < n; c += 32) {
        const int j = c + lane;
        const bool keep = j < n && j <= max_slot && ((s.mask[j] >> warp) & 1u);
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (keep) s.list[warp][cnt + __popc(b & ((1u << lane) - 1u))] = j;
        cnt += __popc(b);
    }
    __syncwarp();
    return cnt;
}

// Forward staging: per splat a 16-bit half-warp mask; per half-warp an ordered slot list.
struct StageFwd {
    float4 xyo[kBatchFwd];
    float4 con[kBatchFwd];
    float4 rgb[kBatchFwd];
    uint16_t mask[kBatchFwd];
    uint16_t list[2 * kWarps][kBatchFwd];
};

template <bool STATS, bool DEPTH, bool FEAT>
__global__ void __launch_bounds__(kThreads) k_raster_fwd(RasterParams p) {
    pdl_trigger();
    pdl_wait();
    __shared__ StageFwd s;
    int tile, cam;
    cta_bin(p, tile, cam);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // warp w: 8x4 block at (8 (w&1), 4 (w>>1)); half h = lane>>4: its left/right 4x4 block
    const int half = lane >> 4, l4 = lane & 15;
    const int hw = 2 * warp + half;   // = 4 * row + column of the 4x4 block
    const int tx = tile % p.TX, ty = tile / p.TX;
    const int px = tx * GS_TILE + (hw & 3) * 4 + (l4 & 3);
    const int py = ty * GS_TILE + (hw >> 2) * 4 + (l4 >> 2);
    const bool inside = px < p.W && py < p.H;
    const float x0 = (float)(tx * GS_TILE), y0 = (float)(ty * GS_TILE);
    const int bin = cam * p.TX * p.TY + tile;
    const int start = p.offs[bin], end = p.offs[bin + 1];

    float T = 1.f, c2 = 0.f, c3 = 0.f, dacc = 0.f;
    float2 c01 = make_float2(0.f, 0.f);   // channels 0, 1: one packed FMA per composite
    int last = start - 1;
    bool done = !inside;
    int n_eval = 0, n_contrib = 0, terminated = 0;
    float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;   // pixel centre
    asm volatile("" : "+f"(fpx), "+f"(fpy));
    const float2 npc = make_float2(-fpx, -fpy);
    const float amax = p.alpha_max, amin = p.alpha_min, tmin = p.t_min;
    const unsigned lt = (1u << lane) - 1u;
    for (int b0 = start; b0 < end; b0 += kBatchFwd) {
        if (__syncthreads_count(done) == kThreads) break;
        const int n = min(kBatchFwd, end - b0);
        for (int t = threadIdx.x; t < n; t += kThreads) {
            const int32_t g = p.ids[b0 + t];
            const float4* rec = reinterpret_cast<const float4*>(p.splats + (int64_t)g * GS_SPLAT_FLOATS);
            const float4 r0 = __ldg(rec), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2);
            s.xyo[t] = r0;
            s.con[t] = prescale_conic(r1.x, r1.y, r1.z);
            s.rgb[t] = FEAT ? load_feat4(p, g, cam) : r2;
            const uint16_t m16 =
                p.cull ? (uint16_t)support_mask16(r0.x, r0.y, r0.z, r1.x, r1.y, r1.z, r1.w, r2.w, x0, y0, amin)
                       : (uint16_t)0xffffu;
            s.mask[t] = m16;
            if (!STATS && p.smask) p.smask[b0 + t] = m16;   // for K7 (every slot K7 can stage is staged here)
        }
        __syncthreads();
        if (__all_sync(0xffffffffu, done)) continue;
        // both half-warp lists of this warp, order preserving
        int cnt0 = 0, cnt1 = 0;
        for (int c = 0; c < n; c += 32) {
            const int j = c + lane;
            const uint32_t m = j < n ? s.mask[j] : 0u;
            const bool k0 = (m >> (2 * warp)) & 1u, k1 = (m >> (2 * warp + 1)) & 1u;
            const unsigned bb0 = __ballot_sync(0xffffffffu, k0), bb1 = __ballot_sync(0xffffffffu, k1);
            if (k0) s.list[2 * warp][cnt0 + __popc(bb0 & lt)] = (uint16_t)j;
            if (k1) s.list[2 * warp + 1][cnt1 + __popc(bb1 & lt)] = (uint16_t)j;
            cnt0 += __popc(bb0);
            cnt1 += __popc(bb1);
        }
        __syncwarp();
        if (done) continue;
        const int cnt = half ? cnt1 : cnt0;
        const uint16_t* list = s.list[hw];
        const uint32_t a_xyo = (uint32_t)__cvta_generic_to_shared(s.xyo);
        const uint32_t a_con = (uint32_t)__cvta_generic_to_shared(s.con);
        const uint32_t a_rgb = (uint32_t)__cvta_generic_to_shared(s.rgb);
        // the two halves of the warp walk their own lists in lockstep; each lane leaves on its
        // own at termination or at the end of its half's list
        int k = 0;
        if (!STATS) {
            // U splats per step: their alphas are evaluated up front (independent LDS / MUFU
            // chains in flight), then composited in list order with predicates instead of
            // branches (a skipped splat changes nothing; a termination stops the rest, Q15), so
            // the result equals the one-at-a-time walk.  Swept on B200: branchy composite U = 1,
            // 2, 3, 4, 6 -> K6 0.246, 0.224, 0.222, 0.220, 0.221 ms; predicated U = 2, 4, 6, 8
            // -> 0.200, 0.198, 0.195, 0.196 ms
#ifndef GS_FWD_UNROLL
#define GS_FWD_UNROLL 6
#endif
            constexpr int U = GS_FWD_UNROLL;
            for (; k + U - 1 < cnt; k += U) {
                uint32_t jj[U];
                float4 xv[U];
                float av[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    jj[u] = (uint32_t)list[k + u] << 4;
                    xv[u] = lds4(a_xyo + jj[u]);
                    float dxu, dyu, Gu;
                    ok[u] = eval_alpha(xv[u].x, xv[u].y, xv[u].z, lds4(a_con + jj[u]), npc, amax, amin, dxu, dyu,
                                       Gu, av[u]);
                }
                bool stop = false;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    // predicated composite: a skipped splat adds exactly 0 (w = 0) and leaves T
                    const bool take = ok[u] && !stop;
                    // (T (1 - alpha) and alpha T as one packed multiply measured slower: the T
                    // recurrence is the walk's serial chain and FMUL2 lengthens it)
                    const float nT = __fmul_rn(T, __fsub_rn(1.f, av[u]));
                    const bool term = take && nT <= tmin;   // Q15: stop without compositing
                    const bool comp = take && !term;
                    const float w = comp ? __fmul_rn(av[u], T) : 0.f;
                    const float4 rgb = lds4(a_rgb + jj[u]);
                    c01 = comp ? fma2(make_float2(rgb.x, rgb.y), bc2(w), c01) : c01;   // 0.190 -> 0.187 ms
                    c2 = comp ? __fmaf_rn(rgb.z, w, c2) : c2;
                    if (FEAT) c3 = comp ? __fmaf_rn(rgb.w, w, c3) : c3;
                    if (DEPTH) dacc = comp ? __fmaf_rn(xv[u].w, w, dacc) : dacc;
                    T = comp ? nT : T;
                    last = comp ? b0 + (int)(jj[u] >> 4) : last;
                    stop = stop || term;
                }
                if (stop) {
                    done = true;
                    break;
                }

            }
            if (done) continue;
        }
        for (; k < cnt; k++) {
            const uint32_t j16 = (uint32_t)list[k] << 4;
            const float4 xyo = lds4(a_xyo + j16);
            float dx, dy, G, alpha;
            if (STATS) n_eval++;
            if (!eval_alpha(xyo.x, xyo.y, xyo.z, lds4(a_con + j16), npc, amax, amin, dx, dy, G, alpha)) continue;
            const float nT = __fmul_rn(T, __fsub_rn(1.f, alpha));
            if (nT <= tmin) {   // Q15: stop without compositing this splat
                done = true;
                if (STATS) terminated = 1;
                break;
            }
            const float w = __fmul_rn(alpha, T);
            const float4 rgb = lds4(a_rgb + j16);
            c01 = fma2(make_float2(rgb.x, rgb.y), bc2(w), c01);   // C += c alpha T
            c2 = __fmaf_rn(rgb.z, w, c2);
            if (FEAT) c3 = __fmaf_rn(rgb.w, w, c3);
            if (DEPTH) dacc = __fmaf_rn(xyo.w, w, dacc);   // sum z alpha T
            T = nT;
            last = b0 + (int)(j16 >> 4);
            if (STATS) n_contrib++;
        }
    }
    const int64_t pix = ((int64_t)cam * p.H + py) * p.W + px;
    if (STATS) {
        if (inside) {
            p.n_eval[pix] = n_eval;
            p.n_contrib[pix] = n_contrib;
            if (p.n_term) p.n_term[pix] = terminated;
        }
        return;
    }
    if (inside && FEAT) {
        const float cc[4] = {c01.x, c01.y, c2, c3};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int ch = p.c0 + k;
            if (ch < p.D) p.out_feats[pix * p.D + ch] = cc[k] + (p.bg ? T * p.bg[cam * p.D + ch] : 0.f);
        }
    }
    if (inside && !FEAT) {
        float g0 = 0.f, g1 = 0.f, g2 = 0.f;
        if (p.bg) {
            g0 = p.bg[3 * cam];
            g1 = p.bg[3 * cam + 1];
            g2 = p.bg[3 * cam + 2];
        }
        p.out_rgb[3 * pix + 0] = c01.x + T * g0;   // R3, Q25
        p.out_rgb[3 * pix + 1] = c01.y + T * g1;
        p.out_rgb[3 * pix + 2] = c2 + T * g2;
    }
    if (inside) {
        p.out_alpha[pix] = 1.f - T;
        p.out_T[pix] = T;
        p.last_ids[pix] = last;
        if (DEPTH) {
            // expected depth: the accumulated depth over sum alpha T = 1 - T_final
            const float A = 1.f - T;
            p.out_depth[pix] = p.depth_mode == 2 ? (A > 0.f ? dacc / A : 0.f) : dacc;
        }
    }
}

// Transposed warp reduction of 8 values: after it, lane l holds the warp sum of value
// (l >> 2) & 7.  9 shuffles + 9 adds instead of 40 + 40.
__device__ __forceinline__ float reduce_scatter8(const float (&v)[8], int lane) {
    // (the stage adds were also tried as packed FADD2 pairs: fewer instructions, but each pair
    // waits for both shuffles -- K7 0.446 -> 0.460 ms)
    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
    float u[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const float send = h4 ? v[i] : v[i + 4];
        const float keep = h4 ? v[i + 4] : v[i];
        u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float w[2];
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const float send = h3 ? u[i] : u[i + 2];
        const float keep = h3 ? u[i + 2] : u[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float x = (h2 ? w[1] : w[0]) + __shfl_xor_sync(0xffffffffu, h2 ? w[0] : w[1], 4);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

// Same for 4 values: lane l holds the warp sum of value (l >> 3) & 3.
__device__ __forceinline__ float reduce_scatter4(const float (&v)[4], int lane) {
    const bool h4 = lane & 16, h3 = lane & 8;
    float u[2];
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const float send = h4 ? v[i] : v[i + 2];
        const float keep = h4 ? v[i + 2] : v[i];
        u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float x = (h3 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, h3 ? u[0] : u[1], 8);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Gradient slots (include/gs.h): 0-7 = the 8-value group (v_mean2d.x, .y, v_opac, v_conic A,
// B, C, v_r, v_g), 8 v_b, 9 v_depth, 10-11 absgrad: the 8-value group is two aligned float4
// (two vector reductions), and the 4-value group (v_b, |v_mean2d.x|, |v_mean2d.y|, v_depth)
// maps to slots {8, 10, 11, 9}.
__device__ __forceinline__ int slot4(int i) { return i == 0 ? 8 : (i == 1 ? 10 : (i == 2 ? 11 : 9)); }

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void red_add_v2(float* addr, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}

#ifndef GS_FEW_LANES
#define GS_FEW_LANES 12
#endif
// <= this many contributing lanes: per-lane vector reductions (measured optimum; 16 before the
// packed FP32x2 gradient block, 11-14 after it: DESIGN.md)
constexpr int kFewLanes = GS_FEW_LANES;

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

#ifdef GS_K7_STATS
// debug builds only (GS_NVCC_EXTRA=-DGS_K7_STATS): visit counters of K7
__device__ unsigned long long g_k7_stats[8];
#define K7_STAT(i, v) \
    do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_k7_stats[i], (unsigned long long)(v)); } while (0)
#else
#define K7_STAT(i, v) do { } while (0)
#endif

template <bool ABSGRAD, bool DEPTH, bool FEAT>
__global__ void __launch_bounds__(kThreads) k_raster_bwd(RasterParams p) {
    pdl_trigger();
    pdl_wait();
    __shared__ Stage<kBatchBwd> s;
    __shared__ int s_maxlast;
    int tile, cam;
    cta_bin(p, tile, cam);
    const PixelCoord q = pixel_coord(p, tile);
    const int bin = cam * p.TX * p.TY + tile;
    const int start = p.offs[bin];
    const int lane = q.lane;

    float Tfin = 1.f, v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, vA = 0.f, bgdot = 0.f, vD = 0.f;
    int last = start - 1;
    if (q.inside) {
        const int64_t pix = ((int64_t)cam * p.H + q.py) * p.W + q.px;
        Tfin = p.out_T[pix];
        last = p.last_ids[pix];
        if (FEAT) {
            // channels [c0, c0+4) of this pass; B4's v_alpha is linear in v_C, so the passes'
            // geometry gradients add up, and the alpha-output term enters in the first pass only
            float vv[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int ch = p.c0 + k;
                vv[k] = ch < p.D ? p.v_feats_img[pix * p.D + ch] : 0.f;
                if (p.bg && ch < p.D) bgdot += p.bg[cam * p.D + ch] * vv[k];
            }
            v0 = vv[0]; v1 = vv[1]; v2 = vv[2]; v3 = vv[3];
            if (p.v_alpha && p.first_pass) vA = p.v_alpha[pix];
        } else {
            v0 = p.v_rgb[3 * pix + 0];
            v1 = p.v_rgb[3 * pix + 1];
            v2 = p.v_rgb[3 * pix + 2];
            if (p.v_alpha) vA = p.v_alpha[pix];
            if (p.bg) bgdot = p.bg[3 * cam] * v0 + p.bg[3 * cam + 1] * v1 + p.bg[3 * cam + 2] * v2;
        }
        if (DEPTH) {
            vD = p.v_depth[pix];
            if (p.depth_mode == 2) {
                // expected depth E = D / A, A = 1 - T_final: dL/dD = v_E / A and, through the
                // alpha output (Q26), dL/dA += -v_E E / A
                const float A = 1.f - Tfin;
                const float vE = vD;
                vD = A > 0.f ? vE / A : 0.f;
                if (A > 0.f) vA -= vE * p.out_depth[pix] / A;
            }
        }
    }
    if (threadIdx.x == 0) s_maxlast = start - 1;
    __syncthreads();
    const int wlast = __reduce_max_sync(0xffffffffu, last);
    if (lane == 0) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int max_last = s_maxlast;
    // constant part of d C_total / d alpha_k: -T_final ra (bg . v_C) + T_final ra v_A (B4)
    const float kbg = Tfin * (vA - bgdot);

    // S only ever enters B4 contracted with this pixel's v_C, so the three channel
    // recurrences are carried as the single scalar Sv = S . v_C (same recurrence, dotted)
    float T = Tfin, Sv = 0.f;
    const float amax = p.alpha_max, amin = p.alpha_min;
    const float2 npc = make_float2(-q.fpx, -q.fpy);   // negated pixel centre (eval_alpha)
    const float2 v01 = make_float2(v0, v1);             // v_C channels 0, 1 as one register pair
    // one (warp, splat) visit: alpha by eval_alpha's operations, B2-B6, the reduction.  tidx is
    // the splat's index in the tile's list (the lane takes it iff tidx <= its last_id)
    auto visit = [&](const float4 xyo, const float4 con, const float4* prgb, const int32_t* pid, int tidx) {
            // the alpha of eval_alpha (same operations, bit-identical decisions as K6), evaluated
            // by every lane without a branch, keeping the products dx^2, dy^2, dx dy for B6: they
            // are finite for any staged record, and a lane that does not take the splat has its
            // G and alpha zeroed below
            const float2 d = add2(make_float2(xyo.x, xyo.y), npc);
            const float2 sq = mul2(d, d);   // dx^2, dy^2
            const float dx = d.x, dy = d.y;
            const float xy = __fmul_rn(dx, dy);
            const float pe = __fmaf_rn(con.z, xy, __fmaf_rn(con.x, sq.x, __fmul_rn(con.y, sq.y)));
            float G = ex2_approx(pe);
            float alpha = fminf(amax, __fmul_rn(xyo.z, G));
            bool valid = q.inside && tidx <= last && !(pe > 0.f) && alpha >= amin;
            const unsigned vb = __ballot_sync(0xffffffffu, valid);
            K7_STAT(0, 1);
            K7_STAT(1, vb == 0);
            K7_STAT(2, __popc(vb));
            K7_STAT(3, (vb != 0) && __popc(vb) <= kFewLanes);
            K7_STAT(4, ((vb & 0xffffu) == 0) != ((vb >> 16) == 0));   // only one 4x4 half takes it
#ifdef GS_K7_STATS
            {   // why lanes idle in non-empty visits: not yet composited (tidx > last) vs outside the support
                const unsigned alive = __ballot_sync(0xffffffffu, q.inside && tidx <= last);
                const unsigned supp = __ballot_sync(0xffffffffu, q.inside && !(pe > 0.f) && alpha >= amin);
                K7_STAT(5, vb ? __popc(alive) : 0);
                K7_STAT(6, vb ? __popc(supp) : 0);
                const unsigned ins = __ballot_sync(0xffffffffu, q.inside);
                K7_STAT(7, vb ? __popc(ins) : 0);
            }
#endif
            if (!vb) return;
            // Branch-free from here: a lane that does not take this splat gets alpha = G = 0,
            // which makes every gradient term below exactly 0 and leaves T and Sv unchanged.
            G = valid ? G : 0.f;
            alpha = valid ? alpha : 0.f;
            float g8[8];   // mx, my, o, A, B, C, r, g
            const float4 rgb = *prgb;
            const float ra = rcp_approx(1.f - alpha);
            T = valid ? T * ra : T;            // B2: T_{n-1} = T_n / (1 - alpha_{n-1})
            const float fac = alpha * T;
            const float2 g67 = mul2(bc2(fac), v01);   // B3: channels 0, 1
            g8[6] = g67.x;
            g8[7] = g67.y;
            const float g_bl = fac * v2;
            const float g_f3 = FEAT ? fac * v3 : 0.f;   // fourth feature channel of the pass
            // B4 + background / alpha-output terms (Q25, Q26):
            // v_alpha = sum_ch (c T - S ra) v_C + kbg ra = T (c . v_C) + ra (kbg - Sv)
            float cv = rgb.x * v0 + rgb.y * v1 + rgb.z * v2;
            if (FEAT) cv += rgb.w * v3;
            float g_z = 0.f;
            if (DEPTH) {                       // depth as a fourth channel
                g_z = fac * vD;
                cv += xyo.w * vD;
            }
            const float v_alpha = T * cv + ra * (kbg - Sv);
            Sv += cv * fac;                    // B5, dotted with v_C
            const float raw = xyo.z * G;
            // B6 (Q24): no gradient through the alpha_max clamp
            const float va = raw < amax ? v_alpha : 0.f;
            g8[2] = G * va;
            const float nvs = raw * va;        // -v_sigma
            const float hv = -0.5f * nvs;      // v_sigma / 2
            g8[3] = hv * sq.x;
            g8[4] = -nvs * xy;
            g8[5] = hv * sq.y;
            // d sigma / d mu' = Sigma'^-1 Delta, with the conic recovered from the
            // pre-scaled one: A = a' (-2 ln2), B = b' (-ln2) = (b'/2)(-2 ln2), C = c' (-2 ln2):
            // (a' dx + (b'/2) dy, c' dy + (b'/2) dx) = (a', c') * d + (b'/2) * swap(d)
            const float2 m = fma2(bc2(con.w), make_float2(dy, dx), mul2(make_float2(con.x, con.y), d));
            const float2 g01 = mul2(bc2((2.f * kLn2) * nvs), m);
            g8[0] = g01.x;
            g8[1] = g01.y;
            const int32_t sid = DEPTH ? *pid : __float_as_int(xyo.w);
            float* dst = p.v_splats + (int64_t)sid * GS_SPLAT_FLOATS;
            if (FEAT) {
                // geometry slots into the record gradient, the 4 channels into v_feats
                float* fdst = p.v_feats + gauss_of(p, sid, cam) * p.D + p.c0;
                const bool ab = ABSGRAD && p.first_pass;
                const int mch = p.D - p.c0;
                if (__popc(vb) <= kFewLanes) {
                    if (valid) {
                        red_add_v4(dst, g8[0], g8[1], g8[2], g8[3]);
                        red_add_v2(dst + 4, g8[4], g8[5]);
                        if (ab) red_add_v2(dst + 10, fabsf(g8[0]), fabsf(g8[1]));
                        atomicAdd(fdst, g8[6]);
                        if (mch > 1) atomicAdd(fdst + 1, g8[7]);
                        if (mch > 2) atomicAdd(fdst + 2, g_bl);
                        if (mch > 3) atomicAdd(fdst + 3, g_f3);
                    }
                    return;
                }
                const float r8 = reduce_scatter8(g8, lane);
                const int i8 = lane >> 2;
                if ((lane & 3) == 0) {
                    if (i8 < 6) atomicAdd(dst + i8, r8);
                    else if (i8 - 6 < mch) atomicAdd(fdst + (i8 - 6), r8);
                }
                const float g4[4] = {g_bl, g_f3, ab ? fabsf(g8[0]) : 0.f, ab ? fabsf(g8[1]) : 0.f};
                const float r4 = reduce_scatter4(g4, lane);
                const int i4 = lane >> 3;
                if ((lane & 7) == 0) {
                    if (i4 < 2) {
                        if (2 + i4 < mch) atomicAdd(fdst + 2 + i4, r4);
                    } else if (ab) {
                        atomicAdd(dst + (i4 == 2 ? 10 : 11), r4);
                    }
                }
                return;
            }
            if (__popc(vb) <= kFewLanes) {
                // few contributing lanes: each issues its own three 16-byte reductions -- 3 warp
                // instructions instead of the ~45 of the shuffle tree
                if (valid) {
                    red_add_v4(dst, g8[0], g8[1], g8[2], g8[3]);
                    red_add_v4(dst + 4, g8[4], g8[5], g8[6], g8[7]);
                    if (ABSGRAD) red_add_v4(dst + 8, g_bl, g_z, fabsf(g8[0]), fabsf(g8[1]));
                    else if (DEPTH) red_add_v2(dst + 8, g_bl, g_z);
                    else atomicAdd(dst + 8, g_bl);
                }
                return;
            }
            const float r8 = reduce_scatter8(g8, lane);
            if ((lane & 3) == 0) atomicAdd(dst + (lane >> 2), r8);
            if (ABSGRAD) {
                const float g4[4] = {g_bl, fabsf(g8[0]), fabsf(g8[1]), g_z};
                const float r4 = reduce_scatter4(g4, lane);
                if ((lane & 7) == 0 && (DEPTH || (lane >> 3) < 3)) atomicAdd(dst + slot4(lane >> 3), r4);
            } else {
                // the ninth value: two folds, then 8 lanes reduce at L2 (3 fewer shuffle + add
                // pairs than the full warp sum; measured 0.466 -> 0.464 ms)
                float rb = g_bl + __shfl_xor_sync(0xffffffffu, g_bl, 16);
                rb += __shfl_xor_sync(0xffffffffu, rb, 8);
                if (lane < 8) atomicAdd(dst + 8, rb);
                if (DEPTH) {
                    const float rz = warp_sum(g_z);
                    if (lane == 0) atomicAdd(dst + 9, rz);
                }
            }
    };
    for (int bend = max_last + 1; bend > start; bend -= kBatchBwd) {
        const int bstart = max(start, bend - kBatchBwd);
        const int n = bend - bstart;
        __syncthreads();
        static_assert(kBatchBwd <= kThreads, "at most one staged splat per thread");
        if ((int)threadIdx.x < n) stage_splat<FEAT, !DEPTH>(p, s, threadIdx.x, bstart + threadIdx.x, q.x0, q.y0, cam);
        __syncthreads();
        if (wlast < bstart) continue;   // warp-uniform: nothing this warp composited here
        const int cnt = build_warp_list(s, n, q.warp, lane, wlast - bstart);
        for (int k = cnt - 1; k >= 0; k--) {
            const int j = s.list[q.warp][k];
            visit(s.xyo[j], s.con[j], &s.rgb[j], &s.id[j], bstart + j);
        }
    }
}

constexpr int kZeroBlocks = 148 * 8;

// Launch order of the backward's (camera, tile) bins: per camera (one block each; the
// cameras stay in sequence, so a camera's records stay hot in L2), its bins in descending
// order of list length -- counting sort on 256 length buckets of 16 intersections -- so the
// longest tiles start first and the launch's tail is made of short ones (the order within a
// bucket is arbitrary: it changes only the fp32 atomic summation order of the gradients).
__global__ void __launch_bounds__(1024) k_tile_order(const int32_t* __restrict__ offs, int TT, int32_t* order) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_cnt[256];
    const int base = blockIdx.x * TT;
    if (threadIdx.x < 256) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < TT; t += 1024) {
        const int len = offs[base + t + 1] - offs[base + t];
        atomicAdd(&s_cnt[255 - min(255, len >> 4)], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the 256 bucket counts, 8 per lane
        const int lane = threadIdx.x;
        int v[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = s_cnt[8 * lane + k];
            sum += v[k];
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int run = x - sum;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            s_cnt[8 * lane + k] = run;
            run += v[k];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < TT; t += 1024) {
        const int len = offs[base + t + 1] - offs[base + t];
        order[base + atomicAdd(&s_cnt[255 - min(255, len >> 4)], 1)] = base + t;
    }
}
#ifndef GS_FWD_PAD
#define GS_FWD_PAD 4096
#endif
constexpr size_t kFwdPad = GS_FWD_PAD;   // dynamic shared-memory pad: at most 4 K6 CTAs per SM
__global__ void __launch_bounds__(256) k_zero4(float4* __restrict__ p, int64_t n4) {
    pdl_trigger();
    pdl_wait();
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n4; i += (int64_t)gridDim.x * 256) p[i] = z;
}

RasterParams make_params(const gs_options& o, int C, int64_t N, int W, int H, const float* splats, const float* bg,
                         const int32_t* ids, const int32_t* offs) {
    RasterParams p{};
    p.C = C; p.W = W; p.H = H; p.N = N;
    p.TX = div_up(W, GS_TILE); p.TY = div_up(H, GS_TILE);
    p.alpha_max = o.alpha_max; p.alpha_min = o.alpha_min; p.t_min = o.t_min;
    p.cull = o.support_cull;
    p.splats = splats; p.bg = bg; p.ids = ids; p.offs = offs;
    return p;
}

}  // namespace

gs_status launch_raster_fwd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats, const float* bg,
                            const int32_t* ids, const int32_t* offs, float* out_rgb, float* out_alpha, float* out_T,
                            int32_t* last_ids, float* out_depth, int depth_mode, uint16_t* isect_masks,
                            cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, bg, ids, offs);
    p.out_rgb = out_rgb; p.out_alpha = out_alpha; p.out_T = out_T; p.last_ids = last_ids;
    p.smask = isect_masks;
    p.out_depth = out_depth; p.depth_mode = out_depth ? depth_mode : 0;
    dim3 grid(p.TX * p.TY, C);
    if (p.depth_mode)
        launch_pdl(k_raster_fwd<false, true, false>, dim3(grid), dim3(kThreads), s, p);
    else
        launch_pdl_smem(k_raster_fwd<false, false, false>, dim3(grid), dim3(kThreads), kFwdPad, s, p);
    GS_LAUNCH_CHECK("k_raster_fwd");
    return GS_OK;
}

gs_status launch_raster_stats(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                              const int32_t* ids, const int32_t* offs, int32_t* n_eval, int32_t* n_contrib,
                              int32_t* terminated, cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, nullptr, ids, offs);
    p.n_eval = n_eval; p.n_contrib = n_contrib; p.n_term = terminated;
    dim3 grid(p.TX * p.TY, C);
    launch_pdl(k_raster_fwd<true, false, false>, dim3(grid), dim3(kThreads), s, p);
    GS_LAUNCH_CHECK("k_raster_fwd<stats>");
    return GS_OK;
}

gs_status launch_raster_bwd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats, const float* bg,
                            const int32_t* ids, const int32_t* offs, const float* out_T, const int32_t* last_ids,
                            const float* v_rgb, const float* v_alpha, const float* out_depth, const float* v_depth,
                            int depth_mode, int absgrad, const uint16_t* isect_masks, const int32_t* tile_order,
                            float* v_splats, cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, bg, ids, offs);
    p.smask = const_cast<uint16_t*>(isect_masks);
    p.out_T = const_cast<float*>(out_T); p.last_ids = const_cast<int32_t*>(last_ids);
    p.v_rgb = v_rgb; p.v_alpha = v_alpha; p.v_splats = v_splats; p.absgrad = absgrad;
    p.out_depth = const_cast<float*>(out_depth); p.v_depth = v_depth;
    p.depth_mode = v_depth ? depth_mode : 0;
    p.order = tile_order;
    const size_t nrec = o.packed ? (size_t)N : (size_t)C * (size_t)N;   // packed: N records in total (Q29)
    // zero-fill as a kernel (not cudaMemsetAsync) so the chain keeps programmatic dependent launch
    if (N > 0 && o.bwd_zero_fill)
        launch_pdl(k_zero4, dim3(kZeroBlocks), dim3(256), s, reinterpret_cast<float4*>(v_splats),
                   (int64_t)(nrec * GS_SPLAT_FLOATS / 4));
    dim3 grid(p.TX * p.TY, C);
    if (absgrad) {
        if (p.depth_mode) launch_pdl(k_raster_bwd<true, true, false>, dim3(grid), dim3(kThreads), s, p);
        else launch_pdl(k_raster_bwd<true, false, false>, dim3(grid), dim3(kThreads), s, p);
    } else {
        if (p.depth_mode) launch_pdl(k_raster_bwd<false, true, false>, dim3(grid), dim3(kThreads), s, p);
        else launch_pdl(k_raster_bwd<false, false, false>, dim3(grid), dim3(kThreads), s, p);
    }
    GS_LAUNCH_CHECK("k_raster_bwd");
    return GS_OK;
}

gs_status launch_zero_splat_grads(float* v_splats, size_t nrec, cudaStream_t s) {
    if (nrec > 0)
        launch_pdl(k_zero4, dim3(kZeroBlocks), dim3(256), s, reinterpret_cast<float4*>(v_splats),
                   (int64_t)(nrec * GS_SPLAT_FLOATS / 4));
    GS_LAUNCH_CHECK("k_zero4");
    return GS_OK;
}

gs_status launch_tile_order(int C, int W, int H, const int32_t* offs, int32_t* order, cudaStream_t s) {
    const int TT = div_up(W, GS_TILE) * div_up(H, GS_TILE);
    launch_pdl(k_tile_order, dim3(C), dim3(1024), s, offs, TT, order);
    GS_LAUNCH_CHECK("k_tile_order");
    return GS_OK;
}

gs_status launch_raster_fwd_nd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                               const float* feats, int D, const int32_t* gids, const float* bg, const int32_t* ids,
                               const int32_t* offs, float* out_feats, float* out_alpha, float* out_T,
                               int32_t* last_ids, uint16_t* isect_masks, cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, bg, ids, offs);
    p.out_alpha = out_alpha; p.out_T = out_T; p.last_ids = last_ids;
    p.smask = isect_masks;
    p.feats = feats; p.D = D; p.gids = gids; p.out_feats = out_feats;
    dim3 grid(p.TX * p.TY, C);
    // channel chunking: 4 channels per pass; every pass composites the same
    // splats (identical T / last_ids / masks)
    for (int c0 = 0; c0 < D; c0 += 4) {
        p.c0 = c0;
        p.first_pass = c0 == 0;
        launch_pdl(k_raster_fwd<false, false, true>, dim3(grid), dim3(kThreads), s, p);
    }
    GS_LAUNCH_CHECK("k_raster_fwd<nd>");
    return GS_OK;
}

gs_status launch_raster_bwd_nd(const gs_options& o, int C, int64_t N, int W, int H, const float* splats,
                               const float* feats, int D, const int32_t* gids, int64_t n_gauss, const float* bg,
                               const int32_t* ids, const int32_t* offs, const float* out_T, const int32_t* last_ids,
                               const float* v_feats_img, const float* v_alpha, int absgrad,
                               const uint16_t* isect_masks, float* v_splats, float* v_feats, cudaStream_t s) {
    RasterParams p = make_params(o, C, N, W, H, splats, bg, ids, offs);
    p.out_T = const_cast<float*>(out_T); p.last_ids = const_cast<int32_t*>(last_ids);
    p.v_alpha = v_alpha; p.v_splats = v_splats; p.absgrad = absgrad;
    p.smask = const_cast<uint16_t*>(isect_masks);
    p.feats = feats; p.D = D; p.gids = gids; p.v_feats_img = v_feats_img; p.v_feats = v_feats;
    const size_t nrec = o.packed ? (size_t)N : (size_t)C * (size_t)N;
    if (N > 0 && o.bwd_zero_fill)
        launch_pdl(k_zero4, dim3(kZeroBlocks), dim3(256), s, reinterpret_cast<float4*>(v_splats),
                   (int64_t)(nrec * GS_SPLAT_FLOATS / 4));
    if (n_gauss > 0 && cudaMemsetAsync(v_feats, 0, sizeof(float) * (size_t)n_gauss * (size_t)D, s) != cudaSuccess) {
        GS_LAUNCH_CHECK("v_feats memset");
        return GS_ERR_CUDA;
    }
    dim3 grid(p.TX * p.TY, C);
    for (int c0 = 0; c0 < D; c0 += 4) {
        p.c0 = c0;
        p.first_pass = c0 == 0;
        if (absgrad)
            launch_pdl(k_raster_bwd<true, false, true>, dim3(grid), dim3(kThreads), s, p);
        else
            launch_pdl(k_raster_bwd<false, false, true>, dim3(grid), dim3(kThreads), s, p);
    }
    GS_LAUNCH_CHECK("k_raster_bwd<nd>");
    return GS_OK;
}

}  // namespace gsb

#ifdef GS_K7_STATS
extern "C" GS_API int gs_debug_k7_stats(unsigned long long* host8, int reset) {
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        return (int)cudaMemcpyToSymbol(gsb::g_k7_stats, z, sizeof z);
    }
    return (int)cudaMemcpyFromSymbol(host8, gsb::g_k7_stats, 8 * sizeof(unsigned long long));
}
#endif
