"""Preallocated execution of the whole hot path through the C-ABI.

`Engine` owns every device buffer of one (N, C, width, height, SH) problem shape and runs
the five stages of include/gs.h on a CUDA stream without any host synchronisation:

    gs_project -> gs_isect_tiles -> gs_rasterize_fwd      (forward)
    gs_rasterize_bwd -> gs_project_bwd                     (backward)

The intersection count M is data dependent.  The engine keeps an M capacity; the
isect stage writes M and an overflow flag on the device, and `ensure_capacity()` (one
small device->host read) grows the capacity and tells the caller to re-run when the
flag is set.  In steady state (bench.py) the flag is checked after the timed region only.
`capture()` records one step into a CUDA graph (every stage is a kernel launch on the
current stream, programmatic dependent launch edges included) and `replay()` re-issues it
with one call: the inputs are read from, and the outputs written to, the same buffers.  With packed=True (Q29) only the visible (camera, Gaussian) pairs
are stored: the projection writes nnz device-side and the per-item buffers are sized by
an nnz capacity handled the same way as M.  Parameter gradients land in ONE flat fp32 buffer (`flat_grad`)
so the data-parallel gradient sum is a single collective.
"""
from __future__ import annotations

import math

import torch

from . import _lib as L
from . import dist as D


class Engine:
    def __init__(self, N, C, width, height, sh_degree=3, K=None, antialiased=False, M_capacity=None,
                 device="cuda", absgrad=False, with_keys=False, packed=False, nnz_capacity=None, depth_mode=0,
                 pose=False, tile_order=True, overlap_prep=True, **opt_kwargs):
        self.N, self.C, self.W, self.H = int(N), int(C), int(width), int(height)
        self.sh_degree = int(sh_degree)
        self.K = (K if K is not None else (self.sh_degree + 1) ** 2) if self.sh_degree >= 0 else 1
        self.absgrad = bool(absgrad)
        self.with_keys = bool(with_keys)
        self.device = torch.device(device)
        self.packed = bool(packed)
        self.depth_mode = int(depth_mode)   # 0 off | 1 accumulated | 2 expected depth
        self.pose = bool(pose)              # camera pose gradients
        self.opts = L.options(sh_degree=self.sh_degree, antialiased=antialiased, packed=self.packed, **opt_kwargs)
        # step(): the backward's preparation -- zero-filling the record gradients, the tile
        # launch order -- runs on a second stream while the forward runs (gs_zero_splat_grads,
        # gs_tile_order), and gs_rasterize_bwd is told not to zero-fill (bwd_zero_fill = 0)
        self.overlap_prep = bool(overlap_prep)
        self._opts_prepped = L.options(sh_degree=self.sh_degree, antialiased=antialiased, packed=self.packed,
                                       bwd_zero_fill=False, **opt_kwargs)
        self.TX, self.TY = L.tiles(self.W, self.H)
        dev = self.device
        C, N, W, H = self.C, self.N, self.W, self.H
        self.nnz = torch.zeros(1, dtype=torch.int64, device=dev)
        self.nnz_overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.nnz_cap = 0
        if self.packed:
            self._alloc_items(nnz_capacity if nnz_capacity is not None else min(C * N, L.MAX_ITEMS))
            pw = L.gs_project_packed_workspace_size(N, C)
            bw = L.gs_project_bwd_packed_workspace_size(N, C)
            self._proj_ws = self._aligned(pw)
            self._pbwd_ws = self._aligned(bw)
        else:
            self.radii = torch.zeros((C, N, 2), dtype=torch.int32, device=dev)
            self.splats = torch.zeros((C, N, L.SPLAT_FLOATS), dtype=torch.float32, device=dev)
            self.v_splats = torch.zeros_like(self.splats)
        self.M = torch.zeros(1, dtype=torch.int64, device=dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.tile_offsets = torch.zeros(C * self.TX * self.TY + 1, dtype=torch.int32, device=dev)
        # launch order of the backward's bins: longest tile lists first (gs_tile_order)
        self.tile_order = torch.zeros(C * self.TX * self.TY, dtype=torch.int32, device=dev) if tile_order else None
        if self.overlap_prep:
            self._side = torch.cuda.Stream(dev)
            self._ev = [torch.cuda.Event() for _ in range(3)]
        self.out_rgb = torch.zeros((C, H, W, 3), dtype=torch.float32, device=dev)
        self.out_alpha = torch.zeros((C, H, W), dtype=torch.float32, device=dev)
        self.out_T = torch.zeros((C, H, W), dtype=torch.float32, device=dev)
        self.last_ids = torch.zeros((C, H, W), dtype=torch.int32, device=dev)
        self.out_depth = torch.zeros((C, H, W), dtype=torch.float32, device=dev) if self.depth_mode else None
        self.v_viewmats = torch.zeros((C, 4, 4), dtype=torch.float32, device=dev) if self.pose else None
        if self.pose and not self.packed:
            self._pbwd_ws = self._aligned(L.gs_project_bwd_workspace_size(N, C))
        elif not self.packed:
            self._pbwd_ws = None
        # flat gradient buffer (the single all-reduce unit, dist.flat_layout)
        sh = self.sh_degree >= 0
        self.flat_layout, total = D.flat_layout(N, self.K, sh)
        self.flat_grad = torch.zeros(total, dtype=torch.float32, device=dev)
        v = D.views(self.flat_grad, N, self.K, sh)
        self.v_quats, self.v_means, self.v_scales = v["quats"], v["means"], v["scales"]
        self.v_opacities, self.v_colors = v["opacities"], v["colors"]
        self.cap = 0
        self.isect_ids = None
        self.isect_keys = None
        self.workspace = None
        self._alloc_isect(M_capacity if M_capacity is not None else max(1 << 16, 4 * C * N))

    # ------------------------------------------------------------------------------
    def _aligned(self, nbytes):
        """A 256-byte aligned uint8 view of nbytes (the C-ABI workspace contract)."""
        raw = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        off = (-raw.data_ptr()) % 256
        return raw[off:off + nbytes]

    def _alloc_items(self, cap):
        """Packed mode: per-item buffers for `cap` visible (camera, Gaussian) pairs."""
        cap = max(int(cap), 1)
        dev = self.device
        self.nnz_cap = cap
        self.radii = torch.zeros((cap, 2), dtype=torch.int32, device=dev)
        self.splats = torch.zeros((cap, L.SPLAT_FLOATS), dtype=torch.float32, device=dev)
        self.v_splats = torch.zeros_like(self.splats)
        self.camera_ids = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.gaussian_ids = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.isect_ids = None   # the isect workspace depends on the item capacity
        self.cap = 0

    @property
    def n_items(self) -> int:
        """Records per call: C*N dense, the packed capacity otherwise (the N of gs_rasterize_*)."""
        return self.nnz_cap if self.packed else self.N

    def _alloc_isect(self, cap):
        cap = int(cap)
        if cap <= self.cap and self.isect_ids is not None:
            return
        self.cap = cap
        self.isect_ids = torch.zeros(max(cap, 1), dtype=torch.int32, device=self.device)
        # per-intersection support masks: written by the forward raster, read by the backward
        self.isect_masks = torch.zeros(max(cap, 1), dtype=torch.int16, device=self.device)
        self.isect_keys = torch.zeros(max(cap, 1), dtype=torch.int64, device=self.device) if self.with_keys else None
        if self.packed:
            ws = L.gs_isect_packed_workspace_size(self.C, self.nnz_cap, self.W, self.H, cap)
        else:
            ws = L.gs_isect_workspace_size(self.C, self.N, self.W, self.H, cap)
        self.workspace_view = self._aligned(ws)

    def ensure_capacity(self, headroom=1.25) -> bool:
        """Reads M and the overflow flag (one D->H sync).  Returns True when the last
        isect overflowed; the capacity is then grown and the caller must re-run."""
        if self.packed and int(self.nnz_overflow.item()) != 0:
            M_cap = self.cap
            nnz = int(self.nnz.item())
            if nnz > L.MAX_ITEMS:
                raise RuntimeError(f"{nnz} visible (camera, Gaussian) pairs exceed the int32 item ids of one call")
            self._alloc_items(min(math.ceil(nnz * headroom) + 1024, L.MAX_ITEMS))
            self._alloc_isect(M_cap)
            return True
        if int(self.overflow.item()) == 0:
            return False
        self._alloc_isect(math.ceil(int(self.M.item()) * headroom) + 1024)
        return True

    def launches_per_step(self) -> int:
        """Kernels of the library launched by one step(): project 1; isect 3 (compaction) +
        3x4 (depth sort) + 3 (tile counts, scan, offsets) + 1 (emission) + 3P (tile sort,
        P = ceil(bits/8)) + 1 (ranges); raster fwd 1; raster bwd 2 (zero-fill + walk) + 1
        (tile order); project bwd 1 (+1 pose reduction).  With overlap_prep the zero-fill and
        the tile order run on the side stream."""
        bits = max(1, (self.C * self.TX * self.TY - 1).bit_length())
        P = (bits + 7) // 8
        pose = 1 if self.pose else 0      # k_pose_reduce
        order = 1 if self.tile_order is not None else 0   # k_tile_order
        if self.packed:   # project: count, scan, write; isect: identity items; project bwd: map + kernel
            return 3 + (1 + 12 + 3 + 1 + 3 * P + 1) + 1 + 2 + order + 2 + pose
        return 1 + (3 + 12 + 3 + 1 + 3 * P + 1) + 1 + 2 + order + 1 + pose

    @property
    def n_isect(self) -> int:
        return int(self.M.item())

    # ------------------------------------------------------------------------------
    def project(self, means, quats, scales, opacities, colors, viewmats, Ks, stream=None):
        if self.packed:
            L.gs_project_packed(self.opts, means, quats, scales, opacities, colors, self.K, viewmats, Ks, self.W,
                                self.H, self.nnz_cap, self.nnz, self.nnz_overflow, self.camera_ids,
                                self.gaussian_ids, self.radii, self.splats, self._proj_ws, stream)
        else:
            L.gs_project(self.opts, means, quats, scales, opacities, colors, self.K, viewmats, Ks, self.W, self.H,
                         self.radii, self.splats, stream)

    def isect(self, stream=None):
        if self.packed:
            L.gs_isect_tiles_packed(self.opts, self.C, self.nnz_cap, self.nnz, self.W, self.H, self.camera_ids,
                                    self.radii, self.splats, self.cap, self.M, self.overflow, self.isect_ids,
                                    self.isect_keys, self.tile_offsets, self.workspace_view, stream)
        else:
            L.gs_isect_tiles(self.opts, self.C, self.N, self.W, self.H, self.radii, self.splats, self.cap, self.M,
                             self.overflow, self.isect_ids, self.isect_keys, self.tile_offsets, self.workspace_view,
                             stream)

    def rasterize_fwd(self, backgrounds=None, stream=None):
        L.gs_rasterize_fwd(self.opts, self.C, self.n_items, self.W, self.H, self.splats, backgrounds,
                           self.isect_ids, self.tile_offsets, self.out_rgb, self.out_alpha, self.out_T,
                           self.last_ids, self.out_depth, self.depth_mode, isect_masks=self.isect_masks,
                           stream=stream)

    def rasterize_bwd(self, v_rgb, v_alpha=None, backgrounds=None, v_depth=None, stream=None, prepped=False):
        """prepped: _prep_begin / _prep_order already zero-filled v_splats and wrote the tile
        order on the side stream (and the caller's stream has waited for them)."""
        if self.tile_order is not None and not prepped:
            L.gs_tile_order(self.opts, self.C, self.W, self.H, self.tile_offsets, self.tile_order, stream)
        L.gs_rasterize_bwd(self._opts_prepped if prepped else self.opts, self.C, self.n_items, self.W, self.H,
                           self.splats, backgrounds,
                           self.isect_ids, self.tile_offsets, self.out_T, self.last_ids, v_rgb, v_alpha,
                           self.absgrad, self.v_splats, out_depth=self.out_depth,
                           v_out_depth=v_depth if self.depth_mode else None, depth_mode=self.depth_mode,
                           isect_masks=self.isect_masks, stream=stream, tile_order=self.tile_order)

    def project_bwd(self, means, quats, scales, opacities, colors, viewmats, Ks, stream=None):
        if self.packed:
            L.gs_project_bwd_packed(self.opts, means, quats, scales, opacities, colors, self.K, viewmats, Ks,
                                    self.W, self.H, self.nnz_cap, self.nnz, self.camera_ids, self.gaussian_ids,
                                    self.radii, self.v_splats, self.v_means, self.v_quats, self.v_scales,
                                    self.v_opacities, self.v_colors, self._pbwd_ws, v_viewmats=self.v_viewmats,
                                    stream=stream)
        else:
            L.gs_project_bwd(self.opts, means, quats, scales, opacities, colors, self.K, viewmats, Ks, self.W,
                             self.H, self.radii, self.v_splats, self.v_means, self.v_quats, self.v_scales,
                             self.v_opacities, self.v_colors, v_viewmats=self.v_viewmats, workspace=self._pbwd_ws,
                             stream=stream)

    def forward(self, means, quats, scales, opacities, colors, viewmats, Ks, backgrounds=None, stream=None):
        self.project(means, quats, scales, opacities, colors, viewmats, Ks, stream)
        self.isect(stream)
        self.rasterize_fwd(backgrounds, stream)

    def backward(self, means, quats, scales, opacities, colors, viewmats, Ks, v_rgb, v_alpha=None,
                 backgrounds=None, v_depth=None, stream=None):
        self.rasterize_bwd(v_rgb, v_alpha, backgrounds, v_depth, stream)
        self.project_bwd(means, quats, scales, opacities, colors, viewmats, Ks, stream)

    def head(self, params, v_rgb, v_alpha=None, backgrounds=None, v_depth=None, stream=None):
        """Everything of step() but the projection backward.  With overlap_prep the record
        gradients are zero-filled on the side stream while the projection and intersection
        run, and the tile order is computed there while the forward composite runs."""
        if not self.overlap_prep:
            self.forward(*params, backgrounds=backgrounds, stream=stream)
            self.rasterize_bwd(v_rgb, v_alpha, backgrounds, v_depth, stream)
            return
        cur = stream if stream is not None else torch.cuda.current_stream(self.device)
        side, ev = self._side, self._ev
        ev[0].record(cur)                 # after the previous reader of v_splats (project_bwd)
        side.wait_event(ev[0])
        L.gs_zero_splat_grads(self.opts, self.C, self.n_items, self.v_splats, side)
        self.project(*params, stream=stream)
        self.isect(stream)
        if self.tile_order is not None:
            ev[1].record(cur)             # tile_offsets written
            side.wait_event(ev[1])
            L.gs_tile_order(self.opts, self.C, self.W, self.H, self.tile_offsets, self.tile_order, side)
        ev[2].record(side)
        self.rasterize_fwd(backgrounds, stream)
        cur.wait_event(ev[2])
        self.rasterize_bwd(v_rgb, v_alpha, backgrounds, v_depth, stream, prepped=True)

    def step(self, params, v_rgb, v_alpha=None, backgrounds=None, v_depth=None, stream=None):
        """One pass of the whole hot path (forward + backward) over one batch of views.
        params = (means, quats, scales, opacities, colors, viewmats, Ks)."""
        self.head(params, v_rgb, v_alpha, backgrounds, v_depth, stream)
        self.project_bwd(*params, stream=stream)

    def capture(self, params, v_rgb, v_alpha=None, backgrounds=None, v_depth=None, head_only=False):
        """Record one step() on these exact tensors into a CUDA graph (the capacities must
        already fit: run run_checked() first).  Returns the graph; replay() launches it.
        head_only: everything but the projection backward (which DPEngine runs in buckets
        interleaved with their all-reduces)."""
        def body():
            if head_only:
                self.head(params, v_rgb, v_alpha, backgrounds, v_depth)
            else:
                self.step(params, v_rgb, v_alpha, backgrounds, v_depth)
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            body()   # warm-up on the capture stream
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        with torch.cuda.graph(self.graph, stream=s):
            body()
        torch.cuda.synchronize(self.device)
        return self.graph

    def replay(self):
        """One captured step (capture()); the overflow flag must be checked as after step()."""
        self.graph.replay()

    def run_checked(self, params, v_rgb, v_alpha=None, backgrounds=None, v_depth=None):
        """step() with capacity growth (syncs once to read the overflow flag)."""
        while True:
            self.step(params, v_rgb, v_alpha, backgrounds, v_depth)
            if not self.ensure_capacity():
                return


class DPEngine(Engine):
    """Views-DP engine whose parameter gradient lives in a bucket-major flat
    buffer (dist.bucket_layout): the projection backward runs bucket by bucket
    (gs_project_bwd_range) and each bucket's all-reduce is issued asynchronously as soon as its
    rows are written, so it overlaps the next bucket's kernel.  Dense layout, no pose."""

    def __init__(self, N, C, width, height, buckets=4, **kw):
        super().__init__(N, C, width, height, **kw)
        if self.packed or self.pose:
            raise ValueError("DPEngine: dense layout without pose gradients")
        sh = self.sh_degree >= 0
        self.bucket_layout, total = D.bucket_layout(self.N, self.K, sh, buckets)
        self.flat_grad = torch.zeros(total, dtype=torch.float32, device=self.device)
        self.buckets = D.bucket_views(self.flat_grad, self.bucket_layout)
        self.v_quats = self.v_means = self.v_scales = self.v_opacities = self.v_colors = None

    def project_bwd(self, means, quats, scales, opacities, colors, viewmats, Ks, stream=None):
        for b in self.buckets:
            self._bucket_bwd(b, (means, quats, scales, opacities, colors, viewmats, Ks), stream)

    def _bucket_bwd(self, b, params, stream=None):
        means, quats, scales, opacities, colors, viewmats, Ks = params
        L.gs_project_bwd_range(self.opts, b["n0"], b["n1"], means, quats, scales, opacities, colors, self.K, viewmats,
                               Ks, self.W, self.H, self.radii, self.v_splats, b["means"], b["quats"], b["scales"],
                               b["opacities"], b["colors"], stream)

    def backward_allreduce(self, params, group=None):
        """The projection backward bucket by bucket, each bucket's gradient summed over the
        group with an asynchronous all-reduce right after its kernel (the collective waits for
        the kernel on the current stream and runs on the process group's stream while the next
        bucket computes); returns after the current stream has waited for every collective."""
        import torch.distributed as dist
        works = []
        for b in self.buckets:
            self._bucket_bwd(b, params)
            works.append(dist.all_reduce(b["flat"], op=dist.ReduceOp.SUM, group=group, async_op=True))
        for w in works:
            w.wait()

    def grads(self):
        """The parameter gradient as full tensors {"v_means": [N,3], ...} (copies)."""
        g = D.gather_buckets(self.flat_grad, self.bucket_layout)
        return {"v_" + k: v for k, v in g.items()}
