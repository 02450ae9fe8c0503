// Stage 2: tile intersection, on-device radix sort, tile ranges -- I1..I4 of SURVEY
// Appendix A, restating App. B.2 of arXiv 2409.06765.
//
// The method orders intersections by (camera, tile, depth) (ties by flat id, Q16).
// Instead of one 48-bit LSD sort over all M intersections, this B200 design sorts in
// two levels, which yields the identical order:
//   1. compact the V visible (c,n) items, in (c,n) order, each with a 16-B record
//      (tile rectangle I1, flat id, camera)                                  [K2a, K2b]
//   2. stable LSD radix sort of the V items by fp32 depth bits (4 x 8 bit)   [K4]
//   3. per sorted item: its record (one gather) and tile count, scan -> M    [K2c, K2d]
//   4. emission of (cam*TT + tile, c*N+n) in depth order, one warp per 32
//      items, coalesced writes                                               [K3]
//   5. stable LSD radix sort of the M pairs by the ceil(log2(C*TT))-bit
//      (camera, tile) key -- 2 passes at 1-MP, <= 15 views                   [K4]
//   6. tile ranges by boundary detection                                     [K5]
// Step 5 being stable keeps step 2's (depth, id) order inside each tile.  Traffic per
// intersection is ~40 B instead of ~144 B for a 6-pass 64-bit sort.  All counts live in
// device memory, so the stage never synchronises the host; grids are sized for the
// capacities and blocks past the live count exit at once.
//
// Radix pass (K4) = three fully parallel kernels (no serial look-back chain, which at
// these sizes -- 0.6 M and 2.9 M keys -- made a single-pass Onesweep latency-bound):
// per-block digit histogram (shared-memory integer atomics), one block per digit scanning
// that digit's row across blocks (coalesced), and a scatter that ranks the block's 1024 keys
// stably in shared memory, reorders them by digit there and writes each digit run with
// consecutive threads.  The scatter's stable warp-level multi-split uses 9 ballots per key.
//
// Compiled with -fmad=false: the tile rectangle (Q20) is evaluated in fp32 with the
// same op order as the oracle so keys match bit for bit.
#include "gs_internal.cuh"

namespace gsb {
namespace {

constexpr int kT = 256;              // threads per block
constexpr int kWarps = kT / 32;
#ifndef GS_VIS_ITEMS
#define GS_VIS_ITEMS 4
#endif
constexpr int kItems = GS_VIS_ITEMS; // compaction: items per thread
constexpr int kTile = kT * kItems;   // compaction: items per block (1024: ~1000 blocks at 1 M items)
constexpr int kSortItems = 4;        // per-item tile counts and small radix sorts: items per thread ...
constexpr int kSortTile = kT * kSortItems;   // ... and per block (1024: enough blocks to fill 148 SMs)
constexpr int kScanThreads = 1024;
#ifndef GS_SCATTER_MATCH
#define GS_SCATTER_MATCH 0
#endif

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// I1 (Q20): half-open tile rectangle [x0,x1) x [y0,y1) in fp32.
__device__ __forceinline__ int4 tile_rect(float mx, float my, int rx, int ry, int TX, int TY) {
    const float ft = (float)GS_TILE;
    int a0 = (int)floorf((mx - (float)rx) / ft), a1 = (int)ceilf((mx + (float)rx) / ft);
    int b0 = (int)floorf((my - (float)ry) / ft), b1 = (int)ceilf((my + (float)ry) / ft);
    return make_int4(clampi(a0, 0, TX), clampi(a1, 0, TX), clampi(b0, 0, TY), clampi(b1, 0, TY));
}

// ---------------------------------------------------------------------------------------
// Block-wide exclusive scan of one int per thread.  Returns the exclusive prefix; *total
// receives the block sum.  s_warp needs 33 ints.
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? s_warp[lane] : 0;
        int wx = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, wx, o);
            if (lane >= o) wx += y;
        }
        if (lane < nw) s_warp[lane] = wx - w;
        if (lane == 31) s_warp[32] = wx;
    }
    __syncthreads();
    int res = x - v + s_warp[warp];
    *total = s_warp[32];
    __syncthreads();
    return res;
}

// Single-block in-place exclusive scan of nb = ceil(n / tile) block sums (n = *d_n or
// n_host, clamped to cap).  Coalesced rounds of 1024.  Writes totals / overflow.
__global__ void __launch_bounds__(kScanThreads) k_scan_blocksums(int* data, int tile, const int* d_n, int64_t n_host,
                                                               int64_t cap, int* total_i32, int64_t* total_i64,
                                                               int32_t* overflow, int64_t ovf_cap, int* clamped_n) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_warp[33];
    const int n = (int)min(d_n ? (int64_t)*d_n : n_host, cap);
    const int nb = div_up(n, tile);
    // the total (M can exceed 2^31 when a call overflows its capacity) is summed in int64; the
    // int32 block offsets saturate just past the capacity, so every position they lead to is
    // >= the clamped count and nothing is emitted there (the overflow flag reports it)
    const int64_t sat = overflow ? min(ovf_cap, (int64_t)INT32_MAX - 1) + 1 : (int64_t)INT32_MAX;
    int64_t carry = 0;
    for (int r = 0; r < nb; r += kScanThreads) {
        const int i = r + threadIdx.x;
        const int v = i < nb ? data[i] : 0;
        int tot;
        const int ex = block_exclusive_scan(v, s_warp, &tot);
        if (i < nb) data[i] = (int)min(carry + ex, sat);
        carry += tot;
    }
    if (threadIdx.x == 0) {
        if (total_i32) *total_i32 = (int)min(carry, (int64_t)INT32_MAX);
        if (total_i64) *total_i64 = carry;
        if (overflow) *overflow = carry > ovf_cap ? 1 : 0;
        if (clamped_n) *clamped_n = (int)min(carry, ovf_cap);
    }
}

struct TileGeom {
    int TX, TY, TT;
    int64_t N;
    const int32_t* cam_ids;   // packed mode: camera of each item (else camera = id / N)
};

// Compact record of a visible item: the packed tile rectangle (Q20) (x0 | x1 << 16,
// y0 | y1 << 16), the flat id (c*N + n, or the packed index) and the camera.  Written in item
// order by the compaction, gathered once per item after the depth sort (16 B instead of the
// 48 B projected record and the radii), so the later stages stream sequentially.
__device__ __forceinline__ int4 compact_record(const float4 r0, int2 r, int32_t id, int cam, const TileGeom& g) {
    const int4 rc = tile_rect(r0.x, r0.y, r.x, r.y, g.TX, g.TY);
    return make_int4(rc.x | (rc.y << 16), rc.z | (rc.w << 16), id, cam);
}

// ---------------------------------------------------------------------------------------
// K2a / K2b: stable compaction of the visible (c,n) items.  Warp w of a block owns the
// contiguous slice [base + 512 w, base + 512 (w+1)) and walks it in 16 coalesced rounds of
// 32; its ballots give every visible item its rank inside the slice without block syncs.
__global__ void __launch_bounds__(kT) k_vis_count(const int2* __restrict__ radii, int64_t n_items, int* blocksum) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_warp[33];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        const int64_t i = base + k * kT + threadIdx.x;
        if (i < n_items) {
            const int2 r = radii[i];
            cnt += (r.x > 0 && r.y > 0) ? 1 : 0;
        }
    }
    int tot;
    block_exclusive_scan(cnt, s_warp, &tot);
    if (threadIdx.x == 0) blocksum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kT) k_vis_compact(const int2* __restrict__ radii, const float* __restrict__ splats,
                                                   int64_t n_items, const int* __restrict__ blockoff, TileGeom g,
                                                   uint32_t* __restrict__ out_key, int32_t* __restrict__ out_val,
                                                   int4* __restrict__ crec) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_wtot[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * kTile + warp * (kTile / kWarps);
    unsigned ball[kItems];
    int run = 0;
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        const int64_t i = base + k * 32 + lane;
        bool vis = false;
        if (i < n_items) {
            const int2 r = radii[i];
            vis = r.x > 0 && r.y > 0;
        }
        ball[k] = __ballot_sync(0xffffffffu, vis);
        run += __popc(ball[k]);
    }
    if (lane == 0) s_wtot[warp] = run;
    __syncthreads();
    int pos = blockoff[blockIdx.x];
    for (int w = 0; w < warp; w++) pos += s_wtot[w];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kItems; k++) {
        if (ball[k] & (1u << lane)) {
            const int64_t i = base + k * 32 + lane;
            const int p = pos + __popc(ball[k] & lt);
            const float4 r0 = reinterpret_cast<const float4*>(splats)[i * 3];   // mu'.x, mu'.y, o, depth
            out_key[p] = __float_as_uint(r0.w);   // depth >= near > 0 (Q17)
            out_val[p] = p;
            crec[p] = compact_record(r0, radii[i], (int32_t)i, (int)(i / g.N), g);
        }
        pos += __popc(ball[k]);
    }
}

// Packed mode: every item is visible, so the "compaction" is the identity on the live
// count V = min(*nnz, cap) (Q29).
__global__ void k_packed_items(const int2* __restrict__ radii, const float* __restrict__ splats, const int64_t* d_nnz,
                               int64_t cap, int* d_V, TileGeom g, uint32_t* __restrict__ out_key,
                               int32_t* __restrict__ out_val, int4* __restrict__ crec) {
    pdl_trigger();
    pdl_wait();
    const int V = (int)min(*d_nnz, cap);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *d_V = V;
    if (i >= V) return;
    const float4 r0 = reinterpret_cast<const float4*>(splats)[i * 3];
    out_key[i] = __float_as_uint(r0.w);
    out_val[i] = (int32_t)i;
    crec[i] = compact_record(r0, radii[i], (int32_t)i, g.cam_ids[i], g);
}

// ---------------------------------------------------------------------------------------
// K4: one stable LSD radix pass (8-bit digit at `shift`), reduce-then-scan.
// hist layout: hist[d * nb_max + b] = count of digit d in block b (digit-major rows).

// Lanes of the warp holding the same 8-bit digit d (d = 256 marks an invalid lane, which
// only matches invalid lanes): 9 ballots.
__device__ __forceinline__ unsigned warp_peers(unsigned d) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; b++) {
        const unsigned bit = (d >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

// digit mask: the compile-time 255 for full 8-bit digits (a runtime mask there cost 8 % of stage
// 2 at configs[2], measured), the runtime one only for the narrower digits of equal-width splits
#define GS_DMASK (NARROW ? mask : 255u)
template <int IT, bool NARROW>
__global__ void __launch_bounds__(kT) k_radix_hist(const uint32_t* __restrict__ keys, const int* d_n, int64_t cap,
                                                   int shift, unsigned mask, int* hist, int nb_max) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_hist[256];
    const int n = (int)min((int64_t)*d_n, cap);
    const int nb = div_up(n, (kT * IT));
    if ((int)blockIdx.x >= nb) return;
    s_hist[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * (kT * IT);
    uint32_t key[IT];
#pragma unroll
    for (int k = 0; k < IT; k++) {
        const int i = base + k * kT + threadIdx.x;
        key[k] = i < n ? keys[i] : 0u;
    }
#pragma unroll
    for (int k = 0; k < IT; k++) {
        const int i = base + k * kT + threadIdx.x;
        const unsigned d = i < n ? (key[k] >> shift) & GS_DMASK : 256u;
        if (d < 256u) atomicAdd(&s_hist[d], 1);
    }
    __syncthreads();
    hist[threadIdx.x * nb_max + blockIdx.x] = s_hist[threadIdx.x];
}

// One block per digit: exclusive scan of that digit's row over the live blocks (each thread
// owns up to kRowItems consecutive entries: one block-wide scan per row); the row total
// goes to rowtot[d].
constexpr int kRowItems = 16;   // rows up to 4096 blocks (4 M keys) in one pass, more in rounds

template <int IT>
__global__ void __launch_bounds__(kT) k_radix_scan_rows(int* hist, int nb_max, const int* d_n, int64_t cap,
                                                        int* rowtot) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_warp[33];
    const int n = (int)min((int64_t)*d_n, cap);
    const int nb = div_up(n, (kT * IT));
    int* row = hist + (int64_t)blockIdx.x * nb_max;
    int carry = 0;
    for (int r = 0; r < nb; r += kT * kRowItems) {
        const int i0 = r + threadIdx.x * kRowItems;
        int v[kRowItems];
        int sum = 0;
#pragma unroll
        for (int k = 0; k < kRowItems; k++) {
            v[k] = i0 + k < nb ? row[i0 + k] : 0;
            sum += v[k];
        }
        int tot;
        int run = carry + block_exclusive_scan(sum, s_warp, &tot);
#pragma unroll
        for (int k = 0; k < kRowItems; k++) {
            if (i0 + k < nb) row[i0 + k] = run;
            run += v[k];
        }
        carry += tot;
    }
    if (threadIdx.x == 0) rowtot[blockIdx.x] = carry;
}

template <int IT, bool NARROW>
__global__ void __launch_bounds__(kT) k_radix_scatter(const uint32_t* __restrict__ keys_in,
                                                      const int32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
                                                      int32_t* __restrict__ vals_out, const int* d_n, int64_t cap,
                                                      int shift, unsigned mask, const int* __restrict__ hist,
                                                      int nb_max, const int* __restrict__ rowtot) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_cnt[kWarps][256];    // per-warp running digit counts, then per-warp offsets
    __shared__ int s_dstart[256];         // start of digit d inside this block's sorted tile
    __shared__ int s_goff[256];           // global start of digit d for this block
    __shared__ int s_warp[33];
    __shared__ uint32_t s_k[(kT * IT)];
    __shared__ int32_t s_v[(kT * IT)];
    const int n = (int)min((int64_t)*d_n, cap);
    const int nb = div_up(n, (kT * IT));
    if ((int)blockIdx.x >= nb) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int w = 0; w < kWarps; w++) s_cnt[w][threadIdx.x] = 0;
    __syncthreads();
    // 1. per-warp stable ranks over the warp's contiguous slice of 128 items
    const int base = blockIdx.x * (kT * IT) + warp * ((kT * IT) / kWarps);
    uint32_t key[IT];
    int32_t val[IT];
    int rank[IT];
#pragma unroll
    for (int k = 0; k < IT; k++) {
        const int i = base + k * 32 + lane;
        const bool valid = i < n;
        key[k] = valid ? keys_in[i] : 0u;
        val[k] = valid ? vals_in[i] : 0;
    }
#pragma unroll
    for (int k = 0; k < IT; k++) {
        const bool valid = base + k * 32 + lane < n;
        const unsigned d = valid ? (key[k] >> shift) & GS_DMASK : 256u;
#if GS_SCATTER_MATCH
        const unsigned peers = __match_any_sync(0xffffffffu, d);
#else
        const unsigned peers = warp_peers(d);
#endif
        int b = 0;
        if (valid) b = s_cnt[warp][d];
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) s_cnt[warp][d] = b + __popc(peers);
        __syncwarp();
        rank[k] = valid ? b + __popc(peers & lt_mask) : -1;
    }
    __syncthreads();
    // 2. per digit: exclusive offsets across warps, block digit totals, digit starts
    {
        const int d = threadIdx.x;
        int run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const int c = s_cnt[w][d];
            s_cnt[w][d] = run;
            run += c;
        }
        int tot;
        s_dstart[d] = block_exclusive_scan(run, s_warp, &tot);   // digits in ascending order
        int dummy;
        s_goff[d] = block_exclusive_scan(rowtot[d], s_warp, &dummy) + hist[d * nb_max + blockIdx.x];
    }
    __syncthreads();
    // 3. reorder the tile by digit in shared memory
#pragma unroll
    for (int k = 0; k < IT; k++) {
        if (rank[k] >= 0) {
            const unsigned d = (key[k] >> shift) & GS_DMASK;
            const int p = s_dstart[d] + s_cnt[warp][d] + rank[k];
            s_k[p] = key[k];
            s_v[p] = val[k];
        }
    }
    __syncthreads();
    // 4. coalesced write-out of the digit runs
    const int nloc = min((kT * IT), n - blockIdx.x * (kT * IT));
#pragma unroll
    for (int k = 0; k < IT; k++) {
        const int j = k * kT + threadIdx.x;
        if (j < nloc) {
            const uint32_t kk = s_k[j];
            const unsigned d = (kk >> shift) & GS_DMASK;
            const int pos = s_goff[d] + (j - s_dstart[d]);
            keys_out[pos] = kk;
            vals_out[pos] = s_v[j];
        }
    }
}

// ---------------------------------------------------------------------------------------
// K2c: tile rectangle and tile count of every depth-sorted visible item (stored for the
// emission), plus per-block (kSortTile items) sums.

__global__ void __launch_bounds__(kT) k_tiles_count(const int4* __restrict__ crec, const int32_t* __restrict__ vis_val,
                                                    const int* d_V, int4* __restrict__ ent_rect,
                                                    int* __restrict__ ent_cnt, int* blocksum) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_warp[33];
    const int V = *d_V;
    const int nb = div_up(V, kSortTile);
    if ((int)blockIdx.x >= nb) return;
    const int base = blockIdx.x * kSortTile;
    int4 e[kSortItems];
#pragma unroll
    for (int k = 0; k < kSortItems; k++) {
        const int j = base + k * kT + threadIdx.x;
        e[k] = j < V ? crec[vis_val[j]] : make_int4(0, 0, 0, 0);
    }
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kSortItems; k++) {
        const int j = base + k * kT + threadIdx.x;
        if (j < V) {
            const int c = ((e[k].x >> 16) - (e[k].x & 0xffff)) * ((e[k].y >> 16) - (e[k].y & 0xffff));
            ent_rect[j] = e[k];
            ent_cnt[j] = c;
            cnt += c;
        }
    }
    int tot;
    block_exclusive_scan(cnt, s_warp, &tot);
    if (threadIdx.x == 0) blocksum[blockIdx.x] = tot;
}

// K2d: exclusive offsets of the per-item counts (ent_off[V] = M), in item order.
__global__ void __launch_bounds__(kT) k_tiles_offsets(const int* __restrict__ ent_cnt, const int* d_V,
                                                      const int* __restrict__ blockoff, int* __restrict__ ent_off) {
    pdl_trigger();
    pdl_wait();
    __shared__ int s_warp[33];
    const int V = *d_V;
    const int nb = div_up(V, kSortTile);
    if ((int)blockIdx.x >= nb) return;
    const int j0 = blockIdx.x * kSortTile + threadIdx.x * kSortItems;
    int c[kSortItems];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kSortItems; k++) {
        c[k] = (j0 + k < V) ? ent_cnt[j0 + k] : 0;
        sum += c[k];
    }
    int tot;
    int run = blockoff[blockIdx.x] + block_exclusive_scan(sum, s_warp, &tot);
#pragma unroll
    for (int k = 0; k < kSortItems; k++) {
        const int j = j0 + k;
        if (j < V) ent_off[j] = run;
        run += c[k];
    }
    if (j0 <= V - 1 && V - 1 < j0 + kSortItems) ent_off[V] = run;   // owner of the last item: run = M
}

// K3 (warp form): each warp emits the intersections of 32 consecutive depth-sorted items.
// The items' offsets sit in the lanes' registers; every output position t of the warp's
// range finds its item by a 5-step binary search over the lanes (shuffles), so the writes
// are coalesced and there is no shared-memory staging or block synchronisation.
__global__ void __launch_bounds__(kT) k_tiles_emit_warp(const int4* __restrict__ ent_rect,
                                                        const int* __restrict__ ent_off, const int* d_V,
                                                        const int* d_nsort, TileGeom g, uint32_t* __restrict__ out_key,
                                                        int32_t* __restrict__ out_val) {
    pdl_trigger();
    pdl_wait();
    const int V = *d_V, n = *d_nsort;
    const int lane = threadIdx.x & 31;
    const int j0 = (blockIdx.x * kT + threadIdx.x) & ~31;   // first item of this warp
    if (j0 >= V) return;
    const int j = j0 + lane;
    const int myoff = ent_off[min(j, V)];                      // ent_off[V] = M (past-the-end)
    const int4 e = j < V ? ent_rect[j] : make_int4(0, 0, 0, 0);
    const int first = __shfl_sync(0xffffffffu, myoff, 0);
    const int end = ent_off[min(j0 + 32, V)];
    const int x0 = e.x & 0xffff, w = (e.x >> 16) - x0, y0 = e.y & 0xffff;
    // key of the item's first tile: an output's key is kbase + qy TX + qx (one shuffle instead
    // of four for camera, x0, y0)
    const uint32_t kbase = (uint32_t)e.w * (uint32_t)g.TT + (uint32_t)(y0 * g.TX + x0);
    const int lim = min(end, n);
    for (int base = first; base < lim; base += 32) {   // warp-uniform trip count
        const int t = base + lane;
        // last lane whose offset is <= t (lanes past V hold M > t)
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int v = __shfl_sync(0xffffffffu, myoff, lo + step);
            if (v <= t) lo += step;
        }
        const int kk = t - __shfl_sync(0xffffffffu, myoff, lo);
        const int ew = __shfl_sync(0xffffffffu, w, lo);
        const uint32_t kb = __shfl_sync(0xffffffffu, kbase, lo);
        const int id = __shfl_sync(0xffffffffu, e.z, lo);
        if (t < lim) {
            // kk / w exactly: kk < w h <= 2^24, so floor((kk + 0.5) / w) survives the fp32 rounding
            const int qy = (int)__fdividef((float)kk + 0.5f, (float)ew);
            out_key[t] = kb + (uint32_t)(qy * g.TX + (kk - qy * ew));
            out_val[t] = id;
        }
    }
}

// K5: tile ranges.  offsets[b] = first sorted index with key >= b; offsets[nbins] = M.
// K5: tile ranges by boundary detection over the sorted keys, 8 keys per thread (two
// 16-byte loads): offsets[b] = first sorted index with key >= b for every b in
// (key[i-1], key[i]], the bins past the last key and all bins of an empty list get n.
constexpr int kRangeKeys = 8;
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys, const int* d_n, int nbins,
                                                int32_t* offsets) {
    pdl_trigger();
    pdl_wait();
    const int n = *d_n;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i0 = t * kRangeKeys;
    if (n == 0) {
        for (int64_t b = t; b <= nbins; b += (int64_t)gridDim.x * blockDim.x) offsets[b] = 0;
        return;
    }
    if (i0 >= n) return;
    uint32_t k[kRangeKeys];
    if (i0 + kRangeKeys <= n) {
        const uint4 a = reinterpret_cast<const uint4*>(keys)[t * 2];
        const uint4 c = reinterpret_cast<const uint4*>(keys)[t * 2 + 1];
        k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = c.x; k[5] = c.y; k[6] = c.z; k[7] = c.w;
    } else {
#pragma unroll
        for (int j = 0; j < kRangeKeys; j++) k[j] = i0 + j < n ? keys[i0 + j] : 0u;
    }
    int64_t prev = i0 > 0 ? (int64_t)keys[i0 - 1] : -1;
#pragma unroll
    for (int j = 0; j < kRangeKeys; j++) {
        if (i0 + j < n) {
            for (int64_t b = prev + 1; b <= (int64_t)k[j]; b++) offsets[b] = (int32_t)(i0 + j);
            prev = k[j];
        }
    }
    if (i0 + kRangeKeys >= n)   // owner of the last key: the bins past it end at n
        for (int64_t b = prev + 1; b <= nbins; b++) offsets[b] = n;
}

__global__ void k_keys64(const uint32_t* __restrict__ keys32, const int32_t* __restrict__ ids,
                         const float* __restrict__ splats, const int* d_n, int TT, int B, uint64_t* out) {
    pdl_trigger();
    pdl_wait();
    const int n = *d_n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys32[i];
    const uint64_t cam = k / (uint32_t)TT, tile = k % (uint32_t)TT;
    const uint32_t dbits = __float_as_uint(splats[(int64_t)ids[i] * GS_SPLAT_FLOATS + 3]);
    out[i] = (cam << (32 + B)) | (tile << 32) | (uint64_t)dbits;
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct WsLayout {
    size_t off_scalars, off_blocksum, off_rowtot, off_hist, off_vk, off_vv, off_ak, off_av, off_rect,
        off_cnt, off_eoff, off_ka, off_va, off_kb, off_vb, off_crec, total;
    int nb_sort_max;   // blocks of kSortTile items (radix passes, tile counts)
};

WsLayout ws_layout(int64_t n_items, int64_t cap) {
    WsLayout L;
    const int64_t big = n_items > cap ? n_items : cap;
    L.nb_sort_max = div_up(big > 0 ? big : 1, kSortTile);
    size_t o = 0;
    L.off_scalars = o; o = align256(o + 64);
    L.off_blocksum = o; o = align256(o + sizeof(int) * (size_t)(L.nb_sort_max + 1));
    L.off_rowtot = o; o = align256(o + sizeof(int) * 256);
    L.off_hist = o; o = align256(o + sizeof(int) * 256 * (size_t)L.nb_sort_max);
    L.off_vk = o; o = align256(o + 4 * (size_t)(n_items + 1));
    L.off_vv = o; o = align256(o + 4 * (size_t)(n_items + 1));
    L.off_ak = o; o = align256(o + 4 * (size_t)(n_items + 1));
    L.off_av = o; o = align256(o + 4 * (size_t)(n_items + 1));
    L.off_rect = o; o = align256(o + 16 * (size_t)(n_items + 1));
    L.off_crec = o; o = align256(o + 16 * (size_t)(n_items + 1));
    L.off_cnt = o; o = align256(o + 4 * (size_t)(n_items + 1));
    L.off_eoff = o; o = align256(o + 4 * (size_t)(n_items + 2));
    L.off_ka = o; o = align256(o + 4 * (size_t)(cap + 1));
    L.off_va = o; o = align256(o + 4 * (size_t)(cap + 1));
    L.off_kb = o; o = align256(o + 4 * (size_t)(cap + 1));
    L.off_vb = o; o = align256(o + 4 * (size_t)(cap + 1));
    L.total = o;
    return L;
}

struct KV {
    uint32_t* k;
    int32_t* v;
};

// ceil(bits/8) stable 8-bit LSD passes over `a` (live count *d_n <= cap), ping-ponging with
// `b`.  The last pass writes its values to `final_vals` when given.  Returns the buffers
// holding the sorted result.
// Keys per block (by the sort's capacity): 1024 below kBigSort keys, 2048 above (half the
// blocks and histogram rows; measured at 14-45 M keys: configs[2] isect 3.69 -> 2.94 ms;
// 4096 was slower at both sizes).  The threshold was 4 M until the shared-memory-atomic
// histograms and equal-width digits; re-swept after them (1, 2, 4 M): configs[1]'s 4 M-capacity
// tile sort is faster with 2048-key blocks (stage 2 0.195 -> 0.187 ms), the 1 M-item depth sort
// gains nothing from them.
#ifndef GS_BIG_SORT_LOG2
#define GS_BIG_SORT_LOG2 21
#endif
constexpr int64_t kBigSort = 1LL << GS_BIG_SORT_LOG2;

template <int IT>
KV radix_sort_t(KV a, KV b, int32_t* final_vals, const int* d_n, int64_t cap, int bits, int* hist, int* rowtot,
                int nb_max, cudaStream_t s) {
    // ceil(bits / 8) passes of (nearly) equal digit width <= 8: e.g. a 13-bit tile key is sorted
    // as 7 + 6 bits rather than 8 + 5 (fewer digits per pass: longer runs in the scatter's
    // coalesced write-out)
    const int passes = bits <= 0 ? 0 : div_up(bits, 8);
    const int width = passes > 0 ? div_up(bits, passes) : 8;   // 13-bit keys: stage 2 0.197 -> 0.195 ms
    const int nb = div_up(cap > 0 ? cap : 1, kT * IT);   // <= nb_max (sized for 1024-key blocks)
    KV in = a, out = b;
    for (int p = 0; p < passes; p++) {
        int32_t* vdst = (p == passes - 1 && final_vals) ? final_vals : out.v;
        const int shift = width * p;
        const unsigned mask = (1u << min(width, bits - shift)) - 1u;
        if (mask == 255u) launch_pdl(k_radix_hist<IT, false>, dim3(nb), dim3(kT), s, in.k, d_n, cap, shift, mask, hist, nb_max);
        else launch_pdl(k_radix_hist<IT, true>, dim3(nb), dim3(kT), s, in.k, d_n, cap, shift, mask, hist, nb_max);
        launch_pdl(k_radix_scan_rows<IT>, dim3(256), dim3(kT), s, hist, nb_max, d_n, cap, rowtot);
        if (mask == 255u)
            launch_pdl(k_radix_scatter<IT, false>, dim3(nb), dim3(kT), s, in.k, in.v, out.k, vdst, d_n, cap, shift, mask,
                       hist, nb_max, rowtot);
        else
            launch_pdl(k_radix_scatter<IT, true>, dim3(nb), dim3(kT), s, in.k, in.v, out.k, vdst, d_n, cap, shift, mask,
                       hist, nb_max, rowtot);
        KV next_in{out.k, vdst};
        out = in;
        in = next_in;
    }
    return in;
}

KV radix_sort(KV a, KV b, int32_t* final_vals, const int* d_n, int64_t cap, int bits, int* hist, int* rowtot,
              int nb_max, cudaStream_t s) {
    if (cap >= kBigSort) return radix_sort_t<8>(a, b, final_vals, d_n, cap, bits, hist, rowtot, nb_max, s);
    return radix_sort_t<4>(a, b, final_vals, d_n, cap, bits, hist, rowtot, nb_max, s);
}

}  // namespace

size_t isect_workspace_bytes(int64_t n_items, int64_t cap) { return ws_layout(n_items, cap).total; }

gs_status launch_isect(const gs_options& o, int C, int64_t N, int W, int H, const int32_t* radii, const float* splats,
                       int64_t n_items, const int64_t* d_nnz, const int32_t* camera_ids, int64_t cap, int64_t* M,
                       int32_t* overflow, int32_t* ids, uint64_t* keys, int32_t* tile_offsets, void* ws,
                       size_t ws_bytes, cudaStream_t s) {
    (void)o;
    const WsLayout L = ws_layout(n_items, cap);
    if (ws_bytes < L.total) return GS_ERR_INVALID_ARGUMENT;
    char* w = static_cast<char*>(ws);
    int* scal = reinterpret_cast<int*>(w + L.off_scalars);
    int* d_V = scal + 0;
    int* d_nsort = scal + 1;
    int* blocksum = reinterpret_cast<int*>(w + L.off_blocksum);
    int* rowtot = reinterpret_cast<int*>(w + L.off_rowtot);
    int* hist = reinterpret_cast<int*>(w + L.off_hist);
    KV vis{reinterpret_cast<uint32_t*>(w + L.off_vk), reinterpret_cast<int32_t*>(w + L.off_vv)};
    KV alt{reinterpret_cast<uint32_t*>(w + L.off_ak), reinterpret_cast<int32_t*>(w + L.off_av)};
    int4* ent_rect = reinterpret_cast<int4*>(w + L.off_rect);
    int4* crec = reinterpret_cast<int4*>(w + L.off_crec);
    int* ent_cnt = reinterpret_cast<int*>(w + L.off_cnt);
    int* ent_off = reinterpret_cast<int*>(w + L.off_eoff);
    KV ia{reinterpret_cast<uint32_t*>(w + L.off_ka), reinterpret_cast<int32_t*>(w + L.off_va)};
    KV ib{reinterpret_cast<uint32_t*>(w + L.off_kb), reinterpret_cast<int32_t*>(w + L.off_vb)};

    const int TX = div_up(W, GS_TILE), TY = div_up(H, GS_TILE), TT = TX * TY;
    const int nbins = C * TT;
    const int B = tile_bits(TT);
    TileGeom g{TX, TY, TT, N > 0 ? N : 1, camera_ids};
    const int2* r2 = reinterpret_cast<const int2*>(radii);
    const int nb_items = div_up(n_items > 0 ? n_items : 1, kTile);

    // 1. stable compaction of the visible (c,n) items (K2a, K2b); identity when packed
    if (d_nnz) {
        launch_pdl(k_packed_items, dim3(div_up(n_items > 0 ? n_items : 1, 256)), dim3(256), s, r2, splats, d_nnz, n_items, d_V,
                   g, vis.k, vis.v, crec);
    } else {
        launch_pdl(k_vis_count, dim3(nb_items), dim3(kT), s, r2, n_items, blocksum);
        launch_pdl(k_scan_blocksums, dim3(1), dim3(kScanThreads), s, blocksum, kTile, nullptr, n_items, INT64_MAX, d_V, nullptr,
                                                     nullptr, 0, nullptr);
        launch_pdl(k_vis_compact, dim3(nb_items), dim3(kT), s, r2, splats, n_items, blocksum, g, vis.k, vis.v, crec);
    }
    GS_LAUNCH_CHECK("isect/compact");
    // 2. stable sort by fp32 depth bits (K4, 4 passes)
    KV dsorted = radix_sort(vis, alt, nullptr, d_V, n_items, 32, hist, rowtot, L.nb_sort_max, s);
    GS_LAUNCH_CHECK("isect/depth-sort");
    // 3. tile rectangles, counts, offsets, M, overflow, clamped count (K2c, K2d)
    const int nb_v = div_up(n_items > 0 ? n_items : 1, kSortTile);
    launch_pdl(k_tiles_count, dim3(nb_v), dim3(kT), s, crec, dsorted.v, d_V, ent_rect, ent_cnt, blocksum);
    launch_pdl(k_scan_blocksums, dim3(1), dim3(kScanThreads), s, blocksum, kSortTile, d_V, 0, INT64_MAX, nullptr, M, overflow, cap,
                                                 d_nsort);
    launch_pdl(k_tiles_offsets, dim3(nb_v), dim3(kT), s, ent_cnt, d_V, blocksum, ent_off);
    // 4. load-balanced emission in depth order (K3)
    if (cap > 0)
        launch_pdl(k_tiles_emit_warp, dim3(div_up(n_items > 0 ? n_items : 1, kT)), dim3(kT), s, ent_rect, ent_off, d_V,
                   d_nsort, g, ia.k, ia.v);
    GS_LAUNCH_CHECK("isect/emit");
    // 5. stable sort by (camera, tile) (K4); values land in the caller's isect_ids
    const int kbits = tile_bits(nbins) > 0 ? tile_bits(nbins) : 1;
    KV sorted = radix_sort(ia, ib, ids, d_nsort, cap, kbits, hist, rowtot, L.nb_sort_max, s);
    GS_LAUNCH_CHECK("isect/tile-sort");
    // 6. tile ranges (K5)
    launch_pdl(k_ranges, dim3(div_up(div_up(cap > 0 ? cap : 1, kRangeKeys), 256)), dim3(256), s, sorted.k, d_nsort,
               nbins, tile_offsets);
    if (keys && cap > 0) launch_pdl(k_keys64, dim3(div_up(cap, 256)), dim3(256), s, sorted.k, sorted.v, splats, d_nsort, TT, B, keys);
    GS_LAUNCH_CHECK("isect/ranges");
    return GS_OK;
}

}  // namespace gsb
