/*
 * gs.h -- C-ABI of libgsplat_b200: the B200 (sm_100a) hot path of the differentiable
 * tile-based 3D Gaussian Splatting rasterizer described in "gsplat: An Open-Source
 * Library for Gaussian Splatting" (arXiv 2409.06765).
 *
 * Citations "P:n" are lines of the paper text; step names F*, I*, R*, B*,
 * P* are SURVEY.md Appendix A, which restates the paper step by step; "Qn" are the
 * readings of ambiguous passages listed in DESIGN.md.
 *
 * The calls follow the paper's user-level statement (Fig. 1)
 *     rgb, alpha, meta = rasterization(means, quats, scales, opacities, colors,
 *                                      viewmats, Ks, width, height)
 * split into the four stages of the method:
 *     gs_project        projection of every (camera, Gaussian)          (App. B.1)
 *     gs_isect_tiles    tile keys, on-device radix sort, tile ranges      (App. B.2)
 *     gs_rasterize_fwd  front-to-back alpha compositing per pixel         (App. B.2)
 *     gs_rasterize_bwd  back-to-front gradient walk per pixel             (App. C.2)
 *     gs_project_bwd    gradients back through the projection             (App. C.3-C.4)
 *
 * CONVENTIONS (all entry points)
 *  - Every array argument is a DEVICE pointer to C-contiguous row-major storage
 *    (fp32 unless stated), 16-byte aligned.  The caller allocates every buffer,
 *    outputs and workspace alike; the library allocates nothing and keeps no mutable
 *    global state (re-entrant, thread-safe).  Ownership never transfers.
 *  - Every call is asynchronous and stream-ordered on `stream` (a cudaStream_t passed
 *    as void*; NULL = the legacy default stream).  No call synchronizes the host.
 *  - Outputs are fully overwritten.  Gradient outputs are zero-filled by the library
 *    before accumulation.
 *  - Argument errors return GS_ERR_INVALID_ARGUMENT (NULL required pointer, N < 0,
 *    C < 1, width/height < 1, misaligned pointer, sh_degree > 3, K < (d+1)^2, too small
 *    workspace); tile_size != 16 returns GS_ERR_UNSUPPORTED; a failed launch returns
 *    GS_ERR_CUDA (gs_last_error() holds the CUDA message, per thread).  Per-element
 *    degeneracies (zero/non-finite quaternion, depth outside [near, far], det <= 0,
 *    off-screen) are never errors: the element is culled (radii = 0).
 *  - Gaussian parameters are ACTIVATED values (scales > 0, opacities in
 *    [0,1]); quaternions (w,x,y,z) need not be normalised (F1 normalises).
 *    Gradients are with respect to the arguments as passed (Q8).
 *  - viewmats [C,4,4] map world to camera (t = W mu + w, Q1), OpenCV axes; Ks [C,3,3]
 *    = [[fx,0,cx],[0,fy,cy],[0,0,1]] (Q2); pixel (i,j) has centre (i+0.5, j+0.5).
 */
#ifndef GSPLAT_B200_GS_H
#define GSPLAT_B200_GS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GS_API __attribute__((visibility("default")))
#else
#define GS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GS_OK = 0,
    GS_ERR_INVALID_ARGUMENT = 1,
    GS_ERR_UNSUPPORTED = 2,
    GS_ERR_CAPACITY = 3,
    GS_ERR_CUDA = 4
} gs_status;

/* Method constants (gs_default_options fills the defaults). */
typedef struct gs_options {
    float near_plane;   /* 0.01  cull iff depth < near (strict; Q18, Fig. 1)          */
    float far_plane;    /* 1e10  cull iff depth > far                                     */
    float eps2d;        /* 0.3   low-pass s added to Sigma' in both modes  */
    float alpha_max;    /* 0.99  opacity saturation (north_star; Q13)                     */
    float alpha_min;    /* 1/255 skip a splat at a pixel iff alpha < alpha_min (Q14)       */
    float t_min;        /* 1e-4  stop iff T(1-alpha) <= t_min, not composited (Q15)        */
    int32_t tile_size;  /* 16 only                                                */
    int32_t antialiased;/* 0 classic | 1 opacity x sqrt(det S'/det(S'+sI))     */
    int32_t sh_degree;  /* -1: colors are RGB [N,3]; 0..3: colors are SH [N,K,3]   */
    int32_t bbox_mode;  /* 0 per-axis 3-sigma AABB (Q12) | 1 square 3 sqrt(lambda_max) |
                           2 opacity-aware: per-axis extent min(3, k(o_eff)) sigma with
                           k^2 = 2 (1.004 tau_ub + 4e-3), tau_ub >= ln(o_eff/alpha_min); o_eff
                           < alpha_min culled (NEXT-4(ii), Q36; images and gradients equal
                           mode 0's, fewer intersections)                              */
    int32_t fov_clamp;  /* 1 clamp t_x/t_z, t_y/t_z to the widened frustum for J only (Q27)*/
    int32_t packed;     /* 0 dense [C,N] records | 1 packed [nnz] records (Q29; the *_packed
                           entry points require 1, the dense ones 0; gs_rasterize_* read
                           N as the total record count when 1)                            */
    int32_t support_cull;/* 1 (default): stages 3/4a skip (splat, 4x4-pixel block) pairs
                           outside the conservative alpha-support of DESIGN.md K6 -- output
                           invariant; 0: evaluate every pair of the tile (verification)   */
    int32_t bwd_zero_fill;/* 1 (default): gs_rasterize_bwd / _nd zero-fill v_splats before
                           accumulating; 0: the caller has zero-filled it (gs_zero_splat_grads,
                           e.g. on a second stream overlapping the forward)              */
} gs_options;

/* ---- Projected splat record ------------------------------------------------------
 * gs_project writes one 48-byte record per (camera c, Gaussian n) at
 * splats[(c*N + n)*GS_SPLAT_FLOATS + k]:
 *   k=0,1  mean2d (mu'_x, mu'_y), pixel coordinates (F11)
 *   k=2    opac_eff = opacity * comp (F15)
 *   k=3    depth = t_z (F4)
 *   k=4..6 conic (A, B, C) = (Sigma' + s I)^-1 = [[A,B],[B,C]] (F10)
 *   k=7    a = (Sigma' + s I)_xx  (blurred variance along x, F8; bounds the alpha support)
 *   k=8..10 rgb (F14)
 *   k=11   c = (Sigma' + s I)_yy
 * Culled records (radii == 0) are all zeros.  gs_rasterize_bwd writes the record
 * GRADIENTS v_splats [.., GS_SPLAT_FLOATS] in their own slot order, chosen so the 8-value
 * group of every (pixel, splat) contribution is two aligned float4 (two vector reductions):
 *   0,1 dL/dmean2d   2 dL/dopac_eff   3,4,5 dL/dconic (A, B, C)   6,7,8 dL/drgb
 *   9 dL/ddepth (0 unless depth rendering)   10,11 absgrad sums |dL/dmean2d| (NEXT-1, 0
 *   unless requested). */
#define GS_SPLAT_FLOATS 12

GS_API void gs_default_options(gs_options* opt);
GS_API const char* gs_status_string(int32_t status);
GS_API const char* gs_last_error(void);     /* last CUDA error text of this thread, "" if none */
GS_API int32_t gs_abi_version(void);         /* = GS_ABI_VERSION */
#define GS_ABI_VERSION 11

/* ---- Stage 1: projection (F1-F15; App. B.1, A.4 P:266-285) ---------------
 * In : means [N,3], quats [N,4] (w,x,y,z), scales [N,3], opacities [N],
 *      colors [N,K,3] (sh_degree >= 0, K >= (d+1)^2) or [N,3] (sh_degree = -1; K ignored;
 *      may be NULL in N-D feature mode, then the record's rgb slots are 0),
 *      viewmats [C,4,4], Ks [C,3,3].
 * Out: radii [C,N,2] int32 (per-axis pixel radius; 0 = culled),
 *      splats [C,N,GS_SPLAT_FLOATS] (record layout above).
 * The fp32 "key path" (mean2d, depth, radii) uses a fixed IEEE op order without FMA
 * contraction (Q28) so tile keys are reproducible bit for bit. */
GS_API gs_status gs_project(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                     const float* means, const float* quats, const float* scales,
                     const float* opacities, const float* colors, int32_t K,
                     const float* viewmats, const float* Ks,
                     int32_t* radii, float* splats, void* stream);

/* ---- Stage 2: tile intersection + on-device radix sort + tile ranges (I1-I4)
 * Each visible (c,n) is binned into every 16x16 tile its 3-sigma rectangle touches
 * (Q20).  The result is ordered by (camera, tile, depth, c*N+n) ascending (Q16).
 * In : radii, splats from gs_project (reads mean2d and depth).
 * Out: *M (device int64)        total number of intersections (may exceed M_capacity;
 *                               summed in int64, so a call whose M passes 2^31 - 1 still
 *                               reports it and sets *overflow: M_capacity < 2^31 - 1)
 *      *overflow (device int32) 1 iff *M > M_capacity (then the outputs are truncated
 *                               and must be recomputed with a larger capacity)
 *      isect_ids [M_capacity]   flat id c*N+n of each intersection, in sorted order
 *      isect_keys [M_capacity]  (optional, NULL to skip) the 64-bit key
 *                               (c << (32+B)) | (tile << 32) | bits(depth_f32),
 *                               B = ceil(log2(TX*TY))
 *      tile_offsets [C*TY*TX+1] int32: intersections of tile t of camera c are
 *                               [tile_offsets[c*TY*TX+t], tile_offsets[c*TY*TX+t+1])
 * workspace: at least gs_isect_workspace_size(C, N, width, height, M_capacity) bytes,
 * 256-byte aligned, contents undefined on entry and exit. */
GS_API size_t gs_isect_workspace_size(int32_t C, int64_t N, int32_t width, int32_t height, int64_t M_capacity);
GS_API gs_status gs_isect_tiles(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                         const int32_t* radii, const float* splats, int64_t M_capacity,
                         int64_t* M, int32_t* overflow, int32_t* isect_ids, uint64_t* isect_keys,
                         int32_t* tile_offsets, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Stage 3: forward composite (R1-R3) ---------------------------------
 * Per pixel p = (i+0.5, j+0.5), front to back over its tile's range:
 *   sigma = 1/2 (A dx^2 + C dy^2) + B dx dy, (dx,dy) = mu' - p; alpha = min(alpha_max,
 *   opac_eff exp(-sigma)); skip alpha < alpha_min; stop when T(1-alpha) <= t_min;
 *   color += rgb alpha T; T *= (1 - alpha).  out = color + T bg.
 * In : splats, isect_ids, tile_offsets; backgrounds [C,3] or NULL (black).
 * Out: out_rgb [C,H,W,3], out_alpha [C,H,W] (= 1 - T), out_T [C,H,W] (final
 *      transmittance, saved for the backward: P:605), last_ids [C,H,W] int32 (index into
 *      isect_ids of the last composited splat; tile_offsets[tile]-1 if none).
 * Depth rendering (App. "Depth rendering"; NULL out_depth = off): out_depth
 *      [C,H,W] = the accumulated depth sum z alpha T (depth_mode 1) or the expected
 *      depth = that sum / sum alpha T, with sum alpha T = 1 - T_final, 0 where nothing was
 *      composited (depth_mode 2); z = record slot 3.  No background term.
 * isect_masks [M] uint16 (optional, NULL to skip): per intersection, the 16-bit mask of the
 *      4x4 pixel blocks of its tile that can take the splat with alpha >= alpha_min (the
 *      conservative support test of DESIGN.md K6; output-invariant).  Pass it to
 *      gs_rasterize_bwd of the same forward to save that kernel recomputing it. */
GS_API gs_status gs_rasterize_fwd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                           const float* splats, const float* backgrounds, const int32_t* isect_ids,
                           const int32_t* tile_offsets, float* out_rgb, float* out_alpha, float* out_T,
                           int32_t* last_ids, float* out_depth, int32_t depth_mode, uint16_t* isect_masks,
                           void* stream);

/* ---- Diagnostics (not on the hot path): per-pixel work counts of stage 3 ---------
 * Runs the forward walk of gs_rasterize_fwd and writes, per pixel, n_eval [C,H,W] (pairs
 * whose alpha was evaluated, up to and including the terminating one) and n_contrib
 * [C,H,W] (pairs composited) and, if non-NULL, terminated [C,H,W] (1 where the walk stopped
 * at the transmittance threshold Q15, 0 where it ran off the end of the tile's list).
 * bench.py uses the sums as the algorithmic work of K6/K7 and the workload descriptors. */
GS_API gs_status gs_rasterize_stats(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                                    const float* splats, const int32_t* isect_ids, const int32_t* tile_offsets,
                                    int32_t* n_eval, int32_t* n_contrib, int32_t* terminated, void* stream);

/* ---- Stage 4a: backward composite (B1-B6) -------------------------------
 * Back to front from last_ids with T_{n-1} = T_n/(1-alpha_{n-1}) and the S
 * recurrence; per-(c,n) sums over pixels are accumulated with fp32 atomics.
 * In : as gs_rasterize_fwd plus out_T, last_ids, v_out_rgb [C,H,W,3],
 *      v_out_alpha [C,H,W] or NULL.
 * Out: v_splats [C,N,GS_SPLAT_FLOATS] ([N,...] when opt->packed; zero-filled here unless
 *      opt->bwd_zero_fill == 0, then accumulated; slot layout above).  absgrad != 0 also accumulates sum |v_mean2d| per pixel into slots 10, 11.
 * Depth (NULL v_out_depth = off): v_out_depth [C,H,W] = dL/d out_depth of the forward
 *      with the same depth_mode; depth is composited as a fourth channel, its per-splat
 *      gradient accumulates into gradient slot 9; mode 2 (expected depth D/A) also needs the
 *      forward's out_depth and adds -v E / A to the alpha gradient (quotient rule, Q26).
 * isect_masks: the forward's mask output or NULL (recomputed).
 * tile_order [C*TY*TX] int32 or NULL: the launch order of the (camera, tile) bins
 *      (gs_tile_order; NULL = camera-major, tile-ascending).  It changes only the order of
 *      the fp32 atomic additions, not the value of any term. */
GS_API gs_status gs_rasterize_bwd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                           const float* splats, const float* backgrounds, const int32_t* isect_ids,
                           const int32_t* tile_offsets, const float* out_T, const int32_t* last_ids,
                           const float* v_out_rgb, const float* v_out_alpha, const float* out_depth,
                           const float* v_out_depth, int32_t depth_mode, int32_t absgrad,
                           const uint16_t* isect_masks, const int32_t* tile_order, float* v_splats,
                           void* stream);

/* ---- Launch order of the backward composite (scheduling only) ---------------------
 * tile_order [C*TY*TX] int32 := every bin c*TY*TX + t of tile_offsets, camera by camera,
 * each camera's tiles in descending order of list length (counting sort on buckets of 16
 * intersections, arbitrary order inside a bucket) -- the longest tiles of the backward
 * start first, so its tail holds short ones.  A permutation of the bins; pass it to
 * gs_rasterize_bwd.  Depends on tile_offsets only. */
GS_API gs_status gs_tile_order(const gs_options* opt, int32_t C, int32_t width, int32_t height,
                               const int32_t* tile_offsets, int32_t* tile_order, void* stream);

/* ---- Zero-fill of the record gradients (scheduling only) ---------------------------
 * v_splats [C,N,GS_SPLAT_FLOATS] ([N,...] when opt->packed) := 0: the zero-fill that
 * gs_rasterize_bwd performs itself unless opt->bwd_zero_fill == 0.  It depends on nothing of
 * the step but the previous reader of v_splats (gs_project_bwd), so a caller can run it on a
 * second stream while the projection and intersection stages run. */
GS_API gs_status gs_zero_splat_grads(const gs_options* opt, int32_t C, int64_t N, float* v_splats, void* stream);

/* ---- Stage 4b: projection backward (P1-P9) -------------------------------
 * In : the gs_project inputs, its radii output, v_splats from gs_rasterize_bwd.
 * Out: v_means [N,3], v_quats [N,4], v_scales [N,3], v_opacities [N],
 *      v_colors (same shape as colors).  Summed over the C cameras inside one thread per
 *      Gaussian (deterministic; Q30); Gaussians culled in every camera get zeros.
 *      Gradient slot 9 of v_splats (dL/d depth, depth rendering) enters through t_z (F4).
 * Pose (NEXT-3; NULL v_viewmats = off): v_viewmats [C,4,4] = dL/d viewmats (App. pose
 *      optimisation): the t = W mu + w, Sigma_c = W Sigma W^T and SH
 *      view-direction (campos = -W^T w) paths; row 3 is 0.  Reduced per (block, camera)
 *      into the workspace (>= gs_project_bwd_workspace_size(N, C) bytes, 256-byte aligned;
 *      unused and may be NULL when v_viewmats is NULL), then summed in block order
 *      (deterministic).
 * v_colors (and colors) may be NULL when sh_degree == -1 (N-D feature mode). */
GS_API size_t gs_project_bwd_workspace_size(int64_t N, int32_t C);

/* ---- Stage 4b over a range of Gaussians (data-parallel gradient buckets) ----
 * gs_project_bwd for the Gaussians [n_begin, n_end) only (0 <= n_begin <= n_end <= N):
 * inputs are the full arrays of gs_project_bwd (means [N,3] ..., radii / v_splats [C,N,...]);
 * the OUTPUTS are the range's own rows -- v_means[(n - n_begin)*3 ...], v_quats, v_scales,
 * v_opacities, v_colors -- so each range can write into its own contiguous bucket and that
 * bucket's all-reduce overlaps the next range's launch.  Per-Gaussian arithmetic, camera sum
 * and results are gs_project_bwd's, bit for bit.  Dense layout; no pose gradients (use
 * gs_project_bwd).  v_colors and colors must be 16-byte aligned for the vector SH path
 * (else the scalar one). */
GS_API gs_status gs_project_bwd_range(const gs_options* opt, int64_t N, int64_t n_begin, int64_t n_end, int32_t C,
                                      int32_t width, int32_t height, const float* means, const float* quats,
                                      const float* scales, const float* opacities, const float* colors, int32_t K,
                                      const float* viewmats, const float* Ks, const int32_t* radii,
                                      const float* v_splats, float* v_means, float* v_quats, float* v_scales,
                                      float* v_opacities, float* v_colors, void* stream);
GS_API gs_status gs_project_bwd(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                         const float* means, const float* quats, const float* scales,
                         const float* opacities, const float* colors, int32_t K,
                         const float* viewmats, const float* Ks, const int32_t* radii,
                         const float* v_splats, float* v_means, float* v_quats, float* v_scales,
                         float* v_opacities, float* v_colors, float* v_viewmats, void* workspace,
                         size_t workspace_bytes, void* stream);

/* ==== N-dimensional features (NEXT-2) =====================================
 * Stage 3 / 4a with D-channel per-Gaussian features feats [n_gauss, D] (camera
 * independent, e.g. learned feature fields) composited exactly like RGB (R1-R3, B1-B6)
 * instead of the record's rgb slots.  Channel chunking: the kernels run once per 4
 * channels (every pass composites the same splats, so out_T / last_ids / isect_masks are
 * those of gs_rasterize_fwd).  Dense: record id c*N+n -> feature row n, gaussian_ids NULL;
 * packed (opt->packed): feature row gaussian_ids[id].  backgrounds: [C, D] or NULL.
 * Out (fwd): out_feats [C,H,W,D], out_alpha, out_T, last_ids, isect_masks as gs_rasterize_fwd.
 * Out (bwd): v_splats (record geometry gradients: slots 0-5; absgrad 10, 11), zero-filled
 *      then accumulated over the passes (B4's v_alpha is linear in v_C; the alpha-output term
 *      enters once), and v_feats [n_gauss, D] = dL/d feats, summed over cameras (zero-filled
 *      here).  For the projection backward of feature mode pass sh_degree = -1 and
 *      v_colors = NULL to gs_project_bwd (its colour gradient is v_feats).
 * Depth rendering is not combined with feature mode (render depth as a feature channel).
 * absgrad != 0 requires D <= 4 (else GS_ERR_UNSUPPORTED): slots 10, 11 hold per-pixel sums of
 * |dL/dmean2d| over ALL channels, which one 4-channel pass sees only when D <= 4. */
GS_API gs_status gs_rasterize_fwd_nd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                                     const float* splats, const float* feats, int32_t D,
                                     const int32_t* gaussian_ids, const float* backgrounds,
                                     const int32_t* isect_ids, const int32_t* tile_offsets, float* out_feats,
                                     float* out_alpha, float* out_T, int32_t* last_ids, uint16_t* isect_masks,
                                     void* stream);
GS_API gs_status gs_rasterize_bwd_nd(const gs_options* opt, int32_t C, int64_t N, int32_t width, int32_t height,
                                     const float* splats, const float* feats, int32_t D,
                                     const int32_t* gaussian_ids, int64_t n_gauss, const float* backgrounds,
                                     const int32_t* isect_ids, const int32_t* tile_offsets, const float* out_T,
                                     const int32_t* last_ids, const float* v_out_feats, const float* v_out_alpha,
                                     int32_t absgrad, const uint16_t* isect_masks, float* v_splats, float* v_feats,
                                     void* stream);

/* ==== Packed mode (Q29; BASELINE configs[4]) ==========================================
 * Only the visible (c,n) pairs are stored: item i of a packed call is the pair
 * (camera_ids[i], gaussian_ids[i]), items ordered camera-major then by Gaussian index,
 * i.e. the order of the visible entries of the dense [C,N] layout.  Every per-item array
 * (radii [nnz,2], splats / v_splats [nnz, GS_SPLAT_FLOATS]) is the dense one with the
 * culled rows removed, so stage 3 / 4a are the SAME calls (gs_rasterize_fwd/bwd with
 * opt->packed = 1 and N = the packed capacity) and their images are bit-identical to the
 * dense path's.  Tile keys are identical; isect_ids hold packed indices instead of c*N+n.
 * The live count nnz stays on the device: the caller sizes nnz_capacity once (e.g. from
 * one read of *nnz, or C*N) and checks *overflow lazily, as for M in stage 2.
 * All three calls require opt->packed == 1. */

/* Projection into the packed layout.  Two passes over the Gaussians (visibility count per
 * (camera, block of 256 Gaussians); scan; full projection writing each visible record at
 * its packed position).  Out: *nnz (device int64), *overflow (device int32: 1 iff *nnz >
 * nnz_capacity; rows past the capacity are dropped), camera_ids / gaussian_ids [cap]
 * int32, radii [cap,2] int32, splats [cap, GS_SPLAT_FLOATS].  Rows >= *nnz are undefined.
 * workspace >= gs_project_packed_workspace_size(N, C) bytes, 256-byte aligned. */
GS_API size_t gs_project_packed_workspace_size(int64_t N, int32_t C);
GS_API gs_status gs_project_packed(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                                   const float* means, const float* quats, const float* scales,
                                   const float* opacities, const float* colors, int32_t K,
                                   const float* viewmats, const float* Ks, int64_t nnz_capacity, int64_t* nnz,
                                   int32_t* overflow, int32_t* camera_ids, int32_t* gaussian_ids, int32_t* radii,
                                   float* splats, void* workspace, size_t workspace_bytes, void* stream);

/* Stage 2 over packed items (nnz read on the device, clamped to nnz_capacity).  Outputs as
 * gs_isect_tiles; isect_ids are packed indices.  workspace >=
 * gs_isect_packed_workspace_size(C, nnz_capacity, width, height, M_capacity). */
GS_API size_t gs_isect_packed_workspace_size(int32_t C, int64_t nnz_capacity, int32_t width, int32_t height,
                                             int64_t M_capacity);
GS_API gs_status gs_isect_tiles_packed(const gs_options* opt, int32_t C, int64_t nnz_capacity, const int64_t* nnz,
                                       int32_t width, int32_t height, const int32_t* camera_ids,
                                       const int32_t* radii, const float* splats, int64_t M_capacity, int64_t* M,
                                       int32_t* overflow, int32_t* isect_ids, uint64_t* isect_keys,
                                       int32_t* tile_offsets, void* workspace, size_t workspace_bytes,
                                       void* stream);

/* Stage 4b from packed per-item gradients v_splats [cap, GS_SPLAT_FLOATS].  Builds the
 * (c,n) -> item map in the workspace (C*N int32), then runs the dense kernel through it:
 * same per-Gaussian camera sum, same outputs as gs_project_bwd.  workspace >=
 * gs_project_bwd_packed_workspace_size(N, C). */
GS_API size_t gs_project_bwd_packed_workspace_size(int64_t N, int32_t C);
GS_API gs_status gs_project_bwd_packed(const gs_options* opt, int64_t N, int32_t C, int32_t width, int32_t height,
                                       const float* means, const float* quats, const float* scales,
                                       const float* opacities, const float* colors, int32_t K,
                                       const float* viewmats, const float* Ks, int64_t nnz_capacity,
                                       const int64_t* nnz, const int32_t* camera_ids, const int32_t* gaussian_ids,
                                       const int32_t* radii, const float* v_splats, float* v_means, float* v_quats,
                                       float* v_scales, float* v_opacities, float* v_colors, float* v_viewmats,
                                       void* workspace, size_t workspace_bytes, void* stream);

/* ==== Gaussian-sharded scale-out ("multi-GPU training support
 * for large-scale scene reconstruction") ===============================================
 * For scenes too large to replicate: rank r of R owns a contiguous shard of the Gaussians
 * and renders a contiguous block of the views, [view_starts[r], view_starts[r+1]).  A step
 * is
 *   owner:  gs_project_packed over its shard and ALL C views  -> items camera-major
 *           gs_shard_pack                                     -> send rows + per-rank counts
 *   NCCL all-to-all of the 16-float rows (views' owners receive, source rank-major)
 *   render: gs_shard_unpack -> gs_isect_tiles_packed / gs_rasterize_fwd / gs_rasterize_bwd
 *           over the received items with C = its own view count
 *   NCCL all-to-all of the per-item v_splats back along the reversed splits
 *   owner:  gs_project_bwd_packed over its shard -> its parameter gradients (no all-reduce).
 * Within each camera the received items are ordered by (source rank, local Gaussian index)
 * = global Gaussian index when shards are contiguous and ascending with rank, so the sort
 * order (camera, tile, depth, item) and hence every image bit equal the one-GPU packed
 * (and dense) call's (Q16, Q29).
 *
 * gs_shard_pack.  In : camera_ids [cap] (camera-major, as gs_project_packed writes them),
 *      *nnz (device, clamped to cap), radii [cap,2], splats [cap, GS_SPLAT_FLOATS], from
 *      gs_project_packed; view_starts: HOST array of R+1 ascending camera indices,
 *      view_starts[0] = 0, view_starts[R] = C; 1 <= R <= 64.
 * Out: send [cap, GS_SHARD_ROW_FLOATS] fp32, row i = item i: the 12 record floats, the two
 *      radii and the destination-local camera id c - view_starts[q] (int32 bit patterns in
 *      floats 12..14), float 15 = 0.  Rows of destination q are contiguous (camera-major).
 *      send_counts [R] int64 (device): rows per destination (sum = min(*nnz, cap)).
 * gs_shard_unpack.  In : recv [n_recv, GS_SHARD_ROW_FLOATS] (host count n_recv).
 * Out: camera_ids [n_recv], radii [n_recv,2], splats [n_recv, GS_SPLAT_FLOATS] and
 *      *nnz = n_recv (device int64), ready for gs_isect_tiles_packed / gs_rasterize_*. */
#define GS_SHARD_ROW_FLOATS 16
GS_API gs_status gs_shard_pack(int64_t nnz_capacity, const int64_t* nnz, int32_t C, int32_t R,
                               const int32_t* view_starts, const int32_t* camera_ids, const int32_t* radii,
                               const float* splats, float* send, int64_t* send_counts, void* stream);
GS_API gs_status gs_shard_unpack(int64_t n_recv, const float* recv, int32_t* camera_ids, int32_t* radii,
                                 float* splats, int64_t* nnz, void* stream);

/* ==== Densification statistics (App. ADC, Absgrad P:204-206)
 * After gs_rasterize_bwd, per Gaussian n over the cameras c where (c,n) is visible
 * (radii > 0), ACCUMULATED IN PLACE (not zero-filled: callers sum over training steps):
 *   grad2d[n]    += || (sx g_x, sy g_y) ||, g = dL/dmu' of that view (v_splats slots 0, 1) or,
 *                   absgrad != 0, its per-pixel absolute sums (slots 10, 11, written by
 *                   gs_rasterize_bwd with absgrad = 1)
 *   count[n]     += 1
 *   max_radii[n]  = max(max_radii[n], max(rx, ry) * radius_scale)   (radius_scale >= 0)
 * Dense (opt->packed == 0): radii [C,N,2], v_splats [C,N,12]; deterministic (one thread per
 * Gaussian sums its cameras in order).  Packed: the per-item rows with gaussian_ids, *nnz
 * clamped to nnz_capacity; fp32 atomics (sum order unspecified).  grad2d, max_radii [N] fp32,
 * count [N] int32. */
GS_API gs_status gs_densify_stats(const gs_options* opt, int64_t N, int32_t C, int64_t nnz_capacity,
                                  const int64_t* nnz, const int32_t* gaussian_ids, const int32_t* radii,
                                  const float* v_splats, int32_t absgrad, float sx, float sy, float radius_scale,
                                  float* grad2d, int32_t* count, float* max_radii, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSPLAT_B200_GS_H */
