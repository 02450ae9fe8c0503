"""Data parallelism over camera views: Gaussians replicated, views partitioned,
parameter gradients summed with ONE all-reduce of a flat fp32 buffer per step.

One process per GPU (torchrun), `torch.distributed` with the NCCL backend on GPUs (gloo in
the CPU tests).  The gradient sum over views equals the gradient of the summed loss
(linearity; Q30), so the R-GPU result equals the 1-GPU result on the same views.
"""
from __future__ import annotations


def partition_views(n_views: int, world: int, rank: int):
    """Contiguous block of view indices for `rank`: view v goes to rank floor(v*R/V)."""
    return [v for v in range(n_views) if (v * world) // n_views == rank]


def _align4(n):
    return (n + 3) // 4 * 4


def flat_layout(N: int, K: int, sh: bool = True):
    """Section offsets (in floats) of the flat gradient buffer:
    [quats 4N | means 3N | scales 3N | opacities N | colors 3KN (SH) or 3N], each section
    16-byte aligned.  Returns (dict name -> (offset, numel, shape), total floats)."""
    ncol = 3 * K * N if sh else 3 * N
    names = ["quats", "means", "scales", "opacities", "colors"]
    sizes = [4 * N, 3 * N, 3 * N, N, ncol]
    shapes = [(N, 4), (N, 3), (N, 3), (N,), (N, K, 3) if sh else (N, 3)]
    out, off = {}, 0
    for n, s, shp in zip(names, sizes, shapes):
        out[n] = (off, s, shp)
        off += _align4(s)
    return out, off


def views(flat, N: int, K: int, sh: bool = True):
    """Named views into a flat gradient tensor."""
    lay, _ = flat_layout(N, K, sh)
    return {n: flat[o:o + s].view(*shp) for n, (o, s, shp) in lay.items()}


def allreduce_grads(flat, group=None):
    """Sum the flat gradient over all ranks (one collective per step)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


def bucket_layout(N: int, K: int, sh: bool = True, n_buckets: int = 4, align: int = 128):
    """Bucket-major layout of the flat gradient for overlapped all-reduce (SURVEY 8(e)
    mitigation 2): bucket b holds the Gaussians [n0, n1) (n0 a multiple of `align`) as
    [quats 4nb | means 3nb | scales 3nb | opacities nb | colors 3K nb], each section 16-byte
    aligned, so each bucket is ONE contiguous all-reduce.  Returns (list of (n0, n1, offset,
    {name: (offset, numel, shape)}), total floats)."""
    per = -(-N // max(1, n_buckets))
    per = -(-per // align) * align if N > 0 else 0
    out, off, n0 = [], 0, 0
    while n0 < N or (N == 0 and not out):
        n1 = min(N, n0 + per) if per else 0
        lay, tot = flat_layout(n1 - n0, K, sh)
        out.append((n0, n1, off, {k: (off + o, s, shp) for k, (o, s, shp) in lay.items()}))
        off += tot
        if n1 == n0:
            break
        n0 = n1
    return out, off


def bucket_views(flat, layout):
    """Per bucket: its flat slice and named section views (one contiguous tensor per bucket)."""
    views_ = []
    for n0, n1, off, secs in layout:
        end = max(o + s for o, s, _ in secs.values()) if secs else off
        d = {n: flat[o:o + s].view(*shp) for n, (o, s, shp) in secs.items()}
        d.update(n0=n0, n1=n1, flat=flat[off:_align4(end)])
        views_.append(d)
    return views_


def gather_buckets(flat, layout):
    """The bucket-major gradient as full per-parameter tensors (copies)."""
    import torch
    vs = bucket_views(flat, layout)
    return {n: torch.cat([v[n] for v in vs]) for n in ["quats", "means", "scales", "opacities", "colors"]}
