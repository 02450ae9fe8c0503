"""Gaussian-sharded scale-out ("multi-GPU training support for
large-scale scene reconstruction").

The views-DP step of `dist.py` replicates every Gaussian on every GPU and all-reduces a
236 B/Gaussian gradient.  For scenes too large to replicate, rank r of R instead OWNS a
contiguous shard of the Gaussians and RENDERS a contiguous block of the views:

    owner   gs_project_packed(shard, all C views)   items camera-major (Q29)
            gs_shard_pack                           16-float rows + rows per destination
    ----    all-to-all #1 (counts), #2 (rows)       NCCL over NVLink / NVSwitch
    render  gs_shard_unpack -> gs_isect_tiles_packed -> gs_rasterize_fwd -> gs_rasterize_bwd
    ----    all-to-all #3: per-item v_splats back along the reversed splits
    owner   gs_project_bwd_packed(shard)            gradients of ITS Gaussians, no all-reduce

Traffic per step is the visible projected records (64 B per visible (camera, Gaussian) item
out, 48 B back) instead of the dense gradient; memory per GPU is N/R Gaussians.  Within a
camera the received items are ordered (source rank, local index) = global Gaussian index,
so the renderer's sort order -- and every image bit -- equals the one-GPU call's (include/gs.h).

Every step of the path runs in the library's kernels (`_lib`); this module allocates buffers
and drives the collectives.  The one host synchronisation per step is the read of the
per-destination row counts that the all-to-all split sizes need.
"""
from __future__ import annotations

import math

import torch

from . import _lib as L
from . import dist as D


def view_starts(n_views: int, world: int):
    """[R+1] first view of each rank under dist.partition_views (contiguous blocks); a rank
    without views starts where the next one does."""
    out = [0] * (world + 1)
    out[world] = n_views
    for q in range(world - 1, -1, -1):
        vs = D.partition_views(n_views, world, q)
        out[q] = vs[0] if vs else out[q + 1]
    return out


def shard_range(n_gauss: int, world: int, rank: int):
    """Contiguous Gaussian shard [n0, n1) of `rank` (ascending with rank, as the ordering
    argument of include/gs.h requires)."""
    return (n_gauss * rank) // world, (n_gauss * (rank + 1)) // world


class Exchange:
    """The two all-to-all patterns of a sharded step over `torch.distributed` (NCCL on GPUs,
    gloo in the CPU tests); world size 1 degenerates to copies."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1

    def counts(self, send_counts: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return send_counts.clone()
        recv = torch.empty_like(send_counts)
        self.dist.all_to_all_single(recv, send_counts, group=self.group)
        return recv

    def rows(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits) -> None:
        if self.world == 1:
            out.copy_(inp)
            return
        self.dist.all_to_all_single(out, inp, list(out_splits), list(in_splits), group=self.group)


class ShardedEngine:
    """One rank's buffers and calls of the Gaussian-sharded step.

    n_local Gaussians (this rank's shard), C views in total (this rank renders
    view_starts[rank]..view_starts[rank+1]).  Phases (each rank runs them in order, the
    exchanges are collective):  project_and_pack -> exchange_forward -> render_forward ->
    render_backward -> exchange_backward -> project_backward.  `step()` runs them all.
    """

    def __init__(self, n_local, C, width, height, rank=0, world=1, sh_degree=3, K=None, antialiased=False,
                 device="cuda", nnz_capacity=None, M_capacity=None, absgrad=False, view_starts=None, recv_capacity=None,
                 **opt_kwargs):
        self.N, self.C, self.W, self.H = int(n_local), int(C), int(width), int(height)
        self.rank, self.world = int(rank), int(world)
        self.sh_degree = int(sh_degree)
        self.K = (K if K is not None else (self.sh_degree + 1) ** 2) if self.sh_degree >= 0 else 1
        self.device = dev = torch.device(device)
        self.absgrad = bool(absgrad)
        self.opts = L.options(sh_degree=self.sh_degree, antialiased=antialiased, packed=True, **opt_kwargs)
        self.vs = list(view_starts) if view_starts is not None else globals()["view_starts"](self.C, self.world)
        if len(self.vs) != self.world + 1 or self.vs[0] != 0 or self.vs[-1] != self.C:
            raise ValueError("view_starts must be [0, ..., C] with one entry per rank + 1")
        self.c0, self.c1 = self.vs[self.rank], self.vs[self.rank + 1]
        self.C_loc = self.c1 - self.c0
        self.TX, self.TY = L.tiles(self.W, self.H)
        # ---- owner side: packed projection of the shard over all C views ----
        self.nnz = torch.zeros(1, dtype=torch.int64, device=dev)
        self.nnz_overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.send_counts = torch.zeros(self.world, dtype=torch.int64, device=dev)
        self._proj_ws = self._aligned(L.gs_project_packed_workspace_size(self.N, self.C))
        self._pbwd_ws = self._aligned(L.gs_project_bwd_packed_workspace_size(self.N, self.C))
        self._alloc_items(nnz_capacity if nnz_capacity is not None else max(1024, self.C * self.N // 2))
        sh = self.sh_degree >= 0
        self.flat_layout, total = D.flat_layout(self.N, self.K, sh)
        self.flat_grad = torch.zeros(total, dtype=torch.float32, device=dev)
        v = D.views(self.flat_grad, self.N, self.K, sh)
        self.v_quats, self.v_means, self.v_scales = v["quats"], v["means"], v["scales"]
        self.v_opacities, self.v_colors = v["opacities"], v["colors"]
        # ---- render side: this rank's views ----
        Cl = max(self.C_loc, 1)
        self.r_nnz = torch.zeros(1, dtype=torch.int64, device=dev)
        self.rcap = 0
        self._alloc_recv(recv_capacity if recv_capacity is not None else self.nnz_cap)
        self.M = torch.zeros(1, dtype=torch.int64, device=dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.tile_offsets = torch.zeros(Cl * self.TX * self.TY + 1, dtype=torch.int32, device=dev)
        H, W = self.H, self.W
        self.out_rgb = torch.zeros((Cl, H, W, 3), dtype=torch.float32, device=dev)
        self.out_alpha = torch.zeros((Cl, H, W), dtype=torch.float32, device=dev)
        self.out_T = torch.zeros((Cl, H, W), dtype=torch.float32, device=dev)
        self.last_ids = torch.zeros((Cl, H, W), dtype=torch.int32, device=dev)
        self.cap = 0
        self._alloc_isect(M_capacity if M_capacity is not None else max(1 << 16, 4 * self.rcap))
        self.n_send = 0
        self.send_splits = [0] * self.world
        self.recv_splits = [0] * self.world
        self.n_recv = 0

    # ------------------------------------------------------------------------------
    def _aligned(self, nbytes):
        raw = torch.empty(int(nbytes) + 256, dtype=torch.uint8, device=self.device)
        off = (-raw.data_ptr()) % 256
        return raw[off:off + int(nbytes)]

    def _alloc_items(self, cap):
        cap = max(int(cap), 1)
        dev = self.device
        self.nnz_cap = cap
        self.camera_ids = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.gaussian_ids = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.radii = torch.zeros((cap, 2), dtype=torch.int32, device=dev)
        self.splats = torch.zeros((cap, L.SPLAT_FLOATS), dtype=torch.float32, device=dev)
        self.v_splats = torch.zeros_like(self.splats)
        self.send = torch.zeros((cap, L.SHARD_ROW_FLOATS), dtype=torch.float32, device=dev)

    def _alloc_recv(self, cap):
        cap = max(int(cap), 1)
        if cap <= self.rcap:
            return False
        dev = self.device
        self.rcap = cap
        self.recv = torch.zeros((cap, L.SHARD_ROW_FLOATS), dtype=torch.float32, device=dev)
        self.r_camera_ids = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.r_radii = torch.zeros((cap, 2), dtype=torch.int32, device=dev)
        self.r_splats = torch.zeros((cap, L.SPLAT_FLOATS), dtype=torch.float32, device=dev)
        self.r_v_splats = torch.zeros_like(self.r_splats)
        return True

    def _alloc_isect(self, cap):
        cap = max(int(cap), 1)
        if cap <= self.cap:
            return
        self.cap = cap
        self.isect_ids = torch.zeros(cap, dtype=torch.int32, device=self.device)
        self.isect_masks = torch.zeros(cap, dtype=torch.int16, device=self.device)
        self._isect_ws_for = None

    def _isect_ws(self):
        key = (self.rcap, self.cap)
        if self._isect_ws_for != key:
            ws = L.gs_isect_packed_workspace_size(max(self.C_loc, 1), self.rcap, self.W, self.H, self.cap)
            self.isect_ws = self._aligned(ws)
            self._isect_ws_for = key
        return self.isect_ws

    # ---- phases ---------------------------------------------------------------------
    def project_and_pack(self, means, quats, scales, opacities, colors, viewmats, Ks, stream=None):
        """Owner: packed projection of the shard over all C views, then the send rows."""
        L.gs_project_packed(self.opts, means, quats, scales, opacities, colors, self.K, viewmats, Ks, self.W,
                            self.H, self.nnz_cap, self.nnz, self.nnz_overflow, self.camera_ids, self.gaussian_ids,
                            self.radii, self.splats, self._proj_ws, stream)
        L.gs_shard_pack(self.nnz_cap, self.nnz, self.C, self.vs, self.camera_ids, self.radii, self.splats, self.send,
                        self.send_counts, stream)

    def read_send_counts(self, headroom=1.25) -> bool:
        """Host read of the per-destination row counts (the step's one sync).  Returns False
        when the shard's nnz overflowed its capacity: buffers are grown and the caller must
        re-run project_and_pack."""
        vals = torch.cat([self.send_counts, self.nnz, self.nnz_overflow.to(torch.int64)]).tolist()
        if vals[-1] != 0:
            self._alloc_items(math.ceil(vals[-2] * headroom) + 1024)
            return False
        self.send_splits = vals[:self.world]
        self.n_send = sum(self.send_splits)
        return True

    def exchange_forward(self, ex: Exchange):
        """All-to-all of the counts, then of the rows (renderer receives source rank-major)."""
        recv_counts = ex.counts(self.send_counts)
        self.recv_splits = recv_counts.tolist()
        self.n_recv = sum(self.recv_splits)
        if self._alloc_recv(math.ceil(self.n_recv * 1.25) + 1024):
            self._alloc_isect(max(self.cap, 4 * self.rcap))
        ex.rows(self.recv[:self.n_recv], self.send[:self.n_send], self.recv_splits, self.send_splits)

    def render_forward(self, backgrounds=None, stream=None):
        """Renderer: unpack, tile intersection and forward composite of its views."""
        L.gs_shard_unpack(self.n_recv, self.recv, self.r_camera_ids, self.r_radii, self.r_splats, self.r_nnz, stream)
        if self.C_loc == 0:
            return
        L.gs_isect_tiles_packed(self.opts, self.C_loc, self.rcap, self.r_nnz, self.W, self.H, self.r_camera_ids,
                                self.r_radii, self.r_splats, self.cap, self.M, self.overflow, self.isect_ids, None,
                                self.tile_offsets, self._isect_ws(), stream)
        L.gs_rasterize_fwd(self.opts, self.C_loc, self.rcap, self.W, self.H, self.r_splats, backgrounds,
                           self.isect_ids, self.tile_offsets, self.out_rgb, self.out_alpha, self.out_T,
                           self.last_ids, isect_masks=self.isect_masks, stream=stream)

    def render_backward(self, v_rgb, v_alpha=None, backgrounds=None, stream=None):
        if self.C_loc == 0:   # no views: nothing was received, nothing goes back
            return
        L.gs_rasterize_bwd(self.opts, self.C_loc, self.rcap, self.W, self.H, self.r_splats, backgrounds,
                           self.isect_ids, self.tile_offsets, self.out_T, self.last_ids, v_rgb, v_alpha,
                           self.absgrad, self.r_v_splats, isect_masks=self.isect_masks, stream=stream)

    def check_isect_capacity(self, headroom=1.25) -> bool:
        """True iff the renderer's intersection buffers overflowed (grown; re-run render_forward)."""
        if self.C_loc == 0 or int(self.overflow.item()) == 0:
            return False
        self._alloc_isect(math.ceil(int(self.M.item()) * headroom) + 1024)
        return True

    def exchange_backward(self, ex: Exchange):
        """All-to-all of the per-item record gradients back to the owners (reversed splits)."""
        ex.rows(self.v_splats[:self.n_send], self.r_v_splats[:self.n_recv], self.send_splits, self.recv_splits)

    def project_backward(self, means, quats, scales, opacities, colors, viewmats, Ks, stream=None):
        L.gs_project_bwd_packed(self.opts, means, quats, scales, opacities, colors, self.K, viewmats, Ks, self.W,
                                self.H, self.nnz_cap, self.nnz, self.camera_ids, self.gaussian_ids, self.radii,
                                self.v_splats, self.v_means, self.v_quats, self.v_scales, self.v_opacities,
                                self.v_colors, self._pbwd_ws, stream=stream)

    def step(self, params, v_rgb, ex: Exchange, v_alpha=None, backgrounds=None):
        """One sharded forward + backward.  params = this rank's (means, quats, scales,
        opacities, colors) shard + ALL (viewmats, Ks); v_rgb [C_loc,H,W,3] for its views.
        Collective: every rank of the group must call it."""
        while True:
            self.project_and_pack(*params)
            if self.read_send_counts():
                break
        self.exchange_forward(ex)
        while True:
            self.render_forward(backgrounds)
            if not self.check_isect_capacity():
                break
        self.render_backward(v_rgb, v_alpha, backgrounds)
        self.exchange_backward(ex)
        self.project_backward(*params)
