"""gsplat (arXiv 2409.06765) hot path, B200-native: differentiable tile-based 3DGS
rasterization as hand-written sm_100a CUDA kernels behind a C-ABI (include/gs.h).

    from paper_2409_06765_b200 import rasterization
    rgb, alpha, meta = rasterization(means, quats, scales, opacities, colors, viewmats, Ks, W, H)
"""
from .rasterization import rasterization  # noqa: F401
from .engine import Engine  # noqa: F401
from . import _lib  # noqa: F401

__all__ = ["rasterization", "Engine"]
