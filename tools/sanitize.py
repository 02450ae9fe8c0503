"""One small run of every library kernel for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): BASELINE configs[0] and a 64k-Gaussian Mip-NeRF-like scene through
the whole step (programmatic-dependent-launch chain included), with depth + pose, absgrad,
packed mode, N-D features, the opacity-aware extent and the support-test-off path, plus
the densification statistics and the shard pack/unpack kernels.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06765_b200 import Engine, rasterization, _lib as L  # noqa: E402
from paper_2409_06765_b200.gshard import ShardedEngine, Exchange  # noqa: E402
from synth import scenes as S  # noqa: E402


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()


def run(sc, **kw):
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v, _ = S.image_grads(0, C, H, W, l1_scale=False)
    params = tuple(t(sc[k]) for k in ["means", "quats", "scales", "opacities", "colors", "viewmats", "Ks"])
    depth = kw.pop("depth_mode", 0)
    eng = Engine(N, C, W, H, sh_degree=sc["sh_degree"], depth_mode=depth, **kw)
    vd = t(np.random.default_rng(0).normal(size=(C, H, W)) * 0.05) if depth else None
    eng.run_checked(params, t(v), None, None, vd)
    torch.cuda.synchronize()
    return eng, params


def main():
    tiny = S.tiny_scene(0)
    mid = S.mipnerf_like_scene(64000, width=320, height=200, views=2, sh_degree=3, seed=3)
    run(tiny)
    eng, _ = run(mid)
    run(mid, depth_mode=2, pose=True, absgrad=True)
    run(mid, packed=True, antialiased=True)
    run(mid, bbox_mode=2)
    run(mid, support_cull=False)
    # diagnostics and statistics kernels
    C, N, W, H = 2, 64000, 320, 200
    ne = torch.zeros((C, H, W), dtype=torch.int32, device="cuda")
    nc, nt = torch.zeros_like(ne), torch.zeros_like(ne)
    L.gs_rasterize_stats(eng.opts, C, eng.n_items, W, H, eng.splats, eng.isect_ids, eng.tile_offsets, ne, nc, nt)
    g2 = torch.zeros(N, device="cuda")
    cnt = torch.zeros(N, dtype=torch.int32, device="cuda")
    mr = torch.zeros(N, device="cuda")
    L.gs_densify_stats(eng.opts, N, C, eng.radii, eng.v_splats, g2, cnt, mr, absgrad=False, scale=(1.0, 1.0),
                       radius_scale=1.0)
    # N-D features through the public API (channel passes)
    sc = dict(mid)
    feats = t(np.random.default_rng(1).normal(size=(N, 5)))
    ts = [t(sc[k]).requires_grad_(True) for k in ["means", "quats", "scales", "opacities"]]
    out, alpha, _ = rasterization(*ts, feats.requires_grad_(True), t(sc["viewmats"]), t(sc["Ks"]), W, H)
    (out.sum() + alpha.sum()).backward()
    # Gaussian-sharded step, one rank (pack -> exchange copies -> unpack)
    se = ShardedEngine(N, C, W, H, rank=0, world=1, sh_degree=3, device="cuda")
    params = tuple(t(mid[k]) for k in ["means", "quats", "scales", "opacities", "colors", "viewmats", "Ks"])
    v, _ = S.image_grads(0, C, H, W, l1_scale=False)
    se.step(params, t(v), Exchange())
    torch.cuda.synchronize()
    print("sanitize run complete")


if __name__ == "__main__":
    main()
